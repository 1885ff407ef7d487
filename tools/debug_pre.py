import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as pkg
from paper_2311_13862_b200 import _native
from oracle import problems as op, solvers as so
spec = pkg.thermal_block((2, 2, 1)); ospec = op.thermal_block((2, 2, 1))
n = int(sys.argv[1]); B = int(sys.argv[2])
prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
oprob = op.OracleProblem(ospec, n, 4)
mus = pkg.sample_mus(spec, B, seed=2000)
ctx = pkg.mg_context_for(prob, mus)
rng = np.random.default_rng(0)
for lvl in range(1, prob.levels):
    nl = prob.cells[lvl]
    x = rng.standard_normal((B, (nl - 1) ** 3)); r = rng.standard_normal((B, (nl - 1) ** 3))
    xt, rt = pkg.to_padded(x, nl), pkg.to_padded(r, nl)
    for mode in range(4):
        y = torch.zeros_like(xt)
        _native.call("rbws_level_kernel", ctx.handle, lvl, mode, xt.data_ptr(), rt.data_ptr(), y.data_ptr(), 0)
        y2 = torch.zeros_like(xt)
        _native.call("rbws_level_kernel", ctx.handle, lvl, mode, xt.data_ptr(), rt.data_ptr(), y2.data_ptr(), 0)
        g = pkg.from_padded(y, nl, B)
        fin = np.isfinite(g).all(axis=1)
        errs = []
        for m in (0, B // 2, B - 1):
            A = oprob.operator(mus[m], level=lvl); d = A.diagonal()
            ref = [A @ x[m], r[m] - A @ x[m], so.jacobi_sweep(A, d, x[m], r[m]),
                   r[m] - A @ (0.7 * r[m] / d)][mode]
            errs.append(float(np.linalg.norm(g[m] - ref) / np.linalg.norm(ref)))
        print("lvl", lvl, "mode", mode, "finite", fin.sum(), "rep", float((y - y2).abs().max()),
              "err", ["%.1e" % e for e in errs], flush=True)
