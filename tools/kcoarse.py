"""Time / profile one level kernel (development tool)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2311_13862_b200 as pkg
from paper_2311_13862_b200 import _native
n, B, lvl, mode, reps = (int(v) for v in sys.argv[1:6])
spec = pkg.thermal_block((2, 2, 1))
prob = pkg.ParametricProblem(spec, levels=pkg.problems.levels_for(n, 4), m0=4)
ctx = pkg.mg_context_for(prob, pkg.sample_mus(spec, B, seed=3))
nl = prob.cells[lvl]
x = torch.randn(pkg.padded_len(nl, B), dtype=torch.float64, device='cuda')
r = torch.randn_like(x); y = torch.zeros_like(x)
f = lambda: _native.call("rbws_level_kernel", ctx.handle, lvl, mode, x.data_ptr(), r.data_ptr(), y.data_ptr(), 0)
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
nodes = B * (nl - 1) ** 3
print(f"level {lvl} n {nl} mode {mode}: {ms:.3f} ms, {nodes/ms/1e6:.1f} Gnode/s, {24*nodes/ms/1e6:.0f} GB/s@24B")
