"""Isolated timing of the fine-level kernels through the C ABI (development tool).

    python tools/kbench.py [--n 64] [--batch 1024] [--reps 5]
"""
import argparse, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2311_13862_b200 as rb
from paper_2311_13862_b200 import _native

ap = argparse.ArgumentParser()
ap.add_argument('--n', type=int, default=64)
ap.add_argument('--batch', type=int, default=1024)
ap.add_argument('--reps', type=int, default=5)
ap.add_argument('--only', default='')
args = ap.parse_args()
n, B = args.n, args.batch
spec = rb.thermal_block((2, 2, 1))
prob = rb.ParametricProblem(spec, levels=rb.problems.levels_for(n, 4), m0=4)
mus = rb.sample_mus(spec, B, seed=3)
ctx = rb.mg_context_for(prob, mus)
L = rb.padded_len(n, B)
x = torch.randn(L, dtype=torch.float64, device='cuda'); y = torch.zeros_like(x)
b = torch.randn(L, dtype=torch.float64, device='cuda'); out = torch.zeros_like(x)
s = torch.cuda.current_stream().cuda_stream
nodes = B * (n - 1) ** 3

def t(name, fn, bytes_per_node):
    if args.only and args.only not in name: return
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    print(f"{name:28s} {ms:8.3f} ms  {bytes_per_node*nodes/ms/1e6:8.1f} GB/s")

t("fine_apply (x->y)", lambda: _native.call("rbws_apply", ctx.handle, prob.finest_level, x.data_ptr(), y.data_ptr(), s), 16)
t("fine_jacobi (x,b->y)", lambda: _native.call("rbws_jacobi_sweep", ctx.handle, prob.finest_level, x.data_ptr(), b.data_ptr(), y.data_ptr(), s), 24)
t("vcycle", lambda: _native.call("rbws_vcycle", ctx.handle, b.data_ptr(), out.data_ptr(), s), 0)
t("copy (torch)", lambda: y.copy_(x), 16)
