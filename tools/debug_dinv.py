import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as pkg
from paper_2311_13862_b200 import _native
from oracle import problems as op
spec = pkg.thermal_block((2, 2, 1)); ospec = op.thermal_block((2, 2, 1))
n = int(sys.argv[1]); B = int(sys.argv[2])
prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
oprob = op.OracleProblem(ospec, n, 4)
mus = pkg.sample_mus(spec, B, seed=2000)
ctx = pkg.mg_context_for(prob, mus)
for lvl in range(1, prob.levels):
    nl = prob.cells[lvl]
    out = torch.zeros(pkg.padded_len(nl, B), dtype=torch.float64, device='cuda')
    _native.call("rbws_batch_dinv", ctx.handle, lvl, out.data_ptr(), 0)
    g = pkg.from_padded(out, nl, B)
    fin = np.isfinite(g).all(axis=1)
    errs = []
    for m in (0, 1, B // 2, B - 1):
        ref = 1.0 / oprob.operator(mus[m], level=lvl).diagonal()
        errs.append(float(np.max(np.abs(g[m] - ref) / np.abs(ref))))
    bad = np.flatnonzero(~fin)
    print("level", lvl, "finite", fin.sum(), "/", B, bad[:5], "relerr", errs, flush=True)
