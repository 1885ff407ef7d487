"""Targeted GPU diagnostics (development tool)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2311_13862_b200 as pkg
from paper_2311_13862_b200 import _native
from oracle import problems as op, solvers as so

def rel(a, b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300)

# 1. prolong with held tensors
ps, os_ = pkg.thermal_block((2,2,1)), op.thermal_block((2,2,1))
prob = pkg.ParametricProblem(ps, levels=3, m0=4); oprob = op.OracleProblem(os_, 16, 4)
P = oprob.prolongations[-1]
rng = np.random.default_rng(1)
rf = rng.standard_normal((2, 15**3)); ec = rng.standard_normal((2, 7**3))
u = pkg.to_padded(rf, 16); e = pkg.to_padded(ec, 8)
torch.cuda.synchronize()
_native.call("rbws_prolong_add", 16, 2, e.data_ptr(), u.data_ptr(), 0); torch.cuda.synchronize()
got = pkg.from_padded(u, 16, 2)
for m in range(2):
    ref = rf[m] + P @ ec[m]; d = np.abs(got[m]-ref)
    bad = np.flatnonzero(d > 1e-12)
    print("prolong", m, rel(got[m], ref), len(bad), [np.unravel_index(b, (15,15,15)) for b in bad[:5]])

# 2. vcycle determinism + per-level for several problems
for case, n, m0 in (((2,2,2), 32, 4), ("smooth", 16, 4), ((2,2,1), 16, 4)):
    if case == "smooth": ps, os_ = pkg.smooth_affine(6), op.smooth_affine(6)
    else: ps, os_ = pkg.thermal_block(case), op.thermal_block(case)
    L = int(np.log2(n//m0))+1
    prob = pkg.ParametricProblem(ps, levels=L, m0=m0); oprob = op.OracleProblem(os_, n, m0)
    mus = op.sample_mus(os_, 2, seed=4)
    ctx = pkg.mg_context_for(prob, mus)
    x = rng.standard_normal((2, (n-1)**3))
    xp = pkg.to_padded(x, n)
    o1 = pkg.mg_vcycle(xp, ctx); o2 = pkg.mg_vcycle(xp, ctx)
    torch.cuda.synchronize()
    print(case, "determinism", float((o1-o2).abs().max()))
    g = pkg.from_padded(o1, n, 2)
    for m in range(2):
        oc = so.mg_context_for(oprob, mus[m])
        print(case, "vcycle vs oracle", m, rel(g[m], so.mg_vcycle(x[m], oc)))
    # dinv at fine level vs oracle diag
    # jacobi per level
    for lvl in range(1, L):
        nl = prob.cells[lvl]
        xx = rng.standard_normal((2, (nl-1)**3)); bb = rng.standard_normal((2, (nl-1)**3))
        xt, bt = pkg.to_padded(xx, nl), pkg.to_padded(bb, nl)
        y = torch.zeros_like(xt)
        _native.call("rbws_jacobi_sweep", ctx.handle, lvl, xt.data_ptr(), bt.data_ptr(), y.data_ptr(), 0)
        torch.cuda.synchronize()
        gy = pkg.from_padded(y, nl, 2)
        errs = []
        for m in range(2):
            A = oprob.operator(mus[m], level=lvl)
            errs.append(rel(gy[m], so.jacobi_sweep(A, A.diagonal(), xx[m], bb[m])))
        print(case, "jacobi level", lvl, errs)
    # mgcg history
    x_, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=30, raise_on_breakdown=False)
    A, f = oprob.operator(mus[0]), oprob.rhs()
    xr, rr = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(oprob, mus[0]), 1e-10, 30)
    print(case, "mgcg iters", [r.iterations for r in reps], rr.iterations)
    print(" gpu hist", np.round(reps[0].history[:6], 8))
    print(" ref hist", np.round(rr.history[:6], 8))
