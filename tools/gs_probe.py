"""Batched MGCG with smoother="gs" vs "jacobi" on the configs[1] shape (development tool)."""
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_2311_13862_b200 as rb

spec = rb.thermal_block((2, 2, 1))
prob = rb.ParametricProblem(spec, levels=5, m0=4)
mus = rb.sample_mus(spec, 1024, seed=5)
for sm in ("jacobi", "gs"):
    ctx = rb.mg_context_for(prob, mus, smoother=sm)
    x, reps = rb.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    torch.cuda.synchronize()
    t = time.perf_counter()
    x, reps = rb.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-10, l_max=60)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    it = reps.iterations
    print(f"{sm:7s} mean iters {it.mean():.2f} max {it.max()}  {dt*1e3:8.1f} ms  {1024/dt:8.1f} solves/s")
