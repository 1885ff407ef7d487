"""example-2 step split (64^3 x 64): mg_context_for (combine + band factorizations) vs
MGCG, live CUDA events."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2311_13862_b200 import fem
from paper_2311_13862_b200.fem_fn import FnFemProblem, mg_context_for, mgcg_solve
from paper_2311_13862_b200.problems import levels_for, lhs_sample

n, batch = 64, 64
spec = fem.example2()
p = FnFemProblem(spec, levels=levels_for(n, 4), m0=4)
mus = np.array(lhs_sample(spec.p, batch, spec.bounds, seed=5))
f = p.rhs(mus)
for _ in range(2):
    ctx = mg_context_for(p, mus)
    mgcg_solve(ctx, f, delta=1e-10, l_max=60)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
ctx = mg_context_for(p, mus)
e[1].record()
x, reps = mgcg_solve(ctx, f, delta=1e-10, l_max=60)
e[2].record()
torch.cuda.synchronize()
print(f"context {e[0].elapsed_time(e[1]):.1f} ms, mgcg {e[1].elapsed_time(e[2]):.1f} ms, "
      f"iterations {reps.iterations.mean():.2f}")
