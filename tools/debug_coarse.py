import os, sys
os.environ["CUDA_LAUNCH_BLOCKING"] = "1"
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as pkg
from paper_2311_13862_b200 import _native
from oracle import problems as op
step = sys.argv[1] if len(sys.argv) > 1 else "all"
ps = pkg.thermal_block((2, 2, 1)); os_ = op.thermal_block((2, 2, 1))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
prob = pkg.ParametricProblem(ps, levels=int(np.log2(n // 4)) + 1, m0=4)
mus = op.sample_mus(os_, 2, seed=1)
print("setup...", flush=True)
ctx = pkg.mg_context_for(prob, mus); torch.cuda.synchronize(); print("setup ok", flush=True)
oprob = op.OracleProblem(os_, n, 4)
for lvl in range(prob.levels):
    nl = prob.cells[lvl]
    x = np.random.default_rng(0).standard_normal((2, (nl - 1) ** 3))
    xt = pkg.to_padded(x, nl)
    y = pkg.BatchOperator(ctx).apply(xt, level=lvl); torch.cuda.synchronize()
    g = pkg.from_padded(y, nl, 2)
    ref = oprob.operator(mus[0], level=lvl) @ x[0]
    print("apply level", lvl, np.linalg.norm(g[0] - ref) / np.linalg.norm(ref), flush=True)
b = torch.randn(pkg.padded_len(n, 2), dtype=torch.float64, device='cuda')
out = pkg.mg_vcycle(b, ctx); torch.cuda.synchronize(); print("vcycle ok", flush=True)
