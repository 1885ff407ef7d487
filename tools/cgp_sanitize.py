"""One batched zero-init MGCG solve at 64^3 with the fused CG update on (37 instances: the
smallest batch the fused kernel takes) — a target for compute-sanitizer memcheck / racecheck.

    compute-sanitizer --tool racecheck python tools/cgp_sanitize.py
"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_13862_b200 as rb
from paper_2311_13862_b200 import _native

n = int(os.environ.get("CGP_N", "64"))
count = int(os.environ.get("CGP_COUNT", "37"))
spec = rb.thermal_block((2, 2, 2))
prob = rb.ParametricProblem(spec, levels=rb.problems.levels_for(n, 4), m0=4)
mus = rb.sample_mus(spec, count, seed=7)
ctx = rb.mg_context_for(prob, mus)
x, reps = rb.mgcg_solve(None, prob.rhs(), None, ctx, delta=1e-6, l_max=int(os.environ.get("CGP_LMAX", "3")))
torch.cuda.synchronize()
print("fused:", bool(_native.load().rbws_batch_cg_fused(ctx.handle)), "iterations", [r.iterations for r in reps][:5])
