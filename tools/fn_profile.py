"""One finest-level plane-block solve of example-2 (64^3, batch 64) for ncu:
ncu -k regex:band_solve -c 1 --set full python tools/fn_profile.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2311_13862_b200 import _native, fem
from paper_2311_13862_b200.fem_fn import FnFemProblem, _ptr, mg_context_for
from paper_2311_13862_b200.problems import levels_for, lhs_sample

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
spec = fem.example2()
p = FnFemProblem(spec, levels=levels_for(n, 4), m0=4)
mus = np.array(lhs_sample(spec.p, batch, spec.bounds, seed=5))
ctx = mg_context_for(p, mus)
r = torch.randn(batch, (n + 1) ** 3, dtype=torch.float64, device="cuda")
x = torch.zeros_like(r)
torch.cuda.synchronize()
_native.call("rbws_fn_band_solve", batch, n, 1, _ptr(ctx.bands[-1]), _ptr(r), _ptr(x), 0.6, 1,
             _native.stream_ptr())
torch.cuda.synchronize()
print("ok")
