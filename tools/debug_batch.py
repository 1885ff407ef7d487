import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as pkg
n = int(sys.argv[1]); B = int(sys.argv[2])
spec = pkg.thermal_block((2, 2, 1))
prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
mus = pkg.sample_mus(spec, B, seed=2000)
ctx = pkg.mg_context_for(prob, mus)
x, reps = pkg.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60, raise_on_breakdown=False)
its = np.array([r.iterations for r in reps]); ok = np.array([r.converged for r in reps])
print("B", B, "iters", np.bincount(its), "converged", ok.sum(), "/", B)
bad = np.flatnonzero(~ok)[:5]
for m in bad: print(" bad", m, mus[m], reps[m].history[:4])
# V-cycle on a random vector: check finiteness per instance
b = torch.randn(pkg.padded_len(n, B), dtype=torch.float64, device='cuda')
o = pkg.mg_vcycle(b, ctx)
fin = torch.isfinite(o[: B * n**3].view(B, -1)).all(dim=1).cpu().numpy()
print("vcycle finite", fin.sum(), "/", B, np.flatnonzero(~fin)[:10])
