"""Per-solve latency of the batched MGCG for several batch sizes (development tool).

    RBWS_GRAPH=0|1 python tools/solve_latency.py
"""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2311_13862_b200 as rb

spec = rb.thermal_block((2, 2, 1))
for n in (32, 64):
    prob = rb.ParametricProblem(spec, levels=rb.problems.levels_for(n, 4), m0=4)
    for B in (1, 8, 64, 256):
        mus = rb.sample_mus(spec, B, seed=5)
        ctx = rb.mg_context_for(prob, mus)
        x0 = torch.zeros(rb.padded_len(n, B), dtype=torch.float64, device="cuda")
        for _ in range(3):
            x, reps = rb.mgcg_solve(None, prob.rhs(), x0, ctx, delta=1e-10, l_max=60)
        torch.cuda.synchronize()
        t = time.perf_counter()
        R = 10
        for _ in range(R):
            x, reps = rb.mgcg_solve(None, prob.rhs(), x0, ctx, delta=1e-10, l_max=60)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / R
        print(f"n={n} batch={B:5d} iters={max(reps.iterations)} {dt*1e3:8.3f} ms/solve-batch "
              f"{B/dt:10.1f} solves/s", flush=True)
