import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as pkg
from paper_2311_13862_b200 import _native
n = 64; B = int(sys.argv[1])
spec = pkg.thermal_block((2, 2, 1))
prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
mus = pkg.sample_mus(spec, B, seed=2000)
ctx = pkg.mg_context_for(prob, mus)
ctx1 = pkg.MgContext(prob, 1)
for lvl in range(prob.levels):
    nl = prob.cells[lvl]
    x = torch.randn(pkg.padded_len(nl, B), dtype=torch.float64, device='cuda')
    blk = x[: B * nl**3].view(B, nl, nl, nl); blk[:, 0] = 0; blk[:, :, 0] = 0; blk[:, :, :, 0] = 0
    x[B * nl**3:] = 0
    y = pkg.BatchOperator(ctx).apply(x, level=lvl)
    bad = []
    for m in (0, 1, 2, 500, 792, B - 1):
        if m >= B: continue
        ctx1.setup(mus[m:m+1])
        x1 = torch.zeros(pkg.padded_len(nl, 1), dtype=torch.float64, device='cuda')
        x1[: nl**3] = x[m * nl**3:(m + 1) * nl**3]
        y1 = pkg.BatchOperator(ctx1).apply(x1, level=lvl)
        d = float((y1[: nl**3] - y[m * nl**3:(m + 1) * nl**3]).abs().max())
        if not d < 1e-12: bad.append((m, d))
    print("level", lvl, "n", nl, "mismatch", bad, flush=True)
