"""Time the finest-level batched apply / residual / Jacobi of example-1 (stored coefficients)
and compare them with the one-node-per-thread kernel (RBWS_FEM_ZM=0 in a second process).

    python tools/fem_apply_bench.py [--n 64] [--batch 256]
"""
import argparse, os, subprocess, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_13862_b200 as rb
from paper_2311_13862_b200 import _native

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--child", action="store_true")
args = ap.parse_args()
n, B = args.n, args.batch
spec = rb.get_problem("example-1")
prob = rb.ParametricProblem(spec, levels=rb.problems.levels_for(n, 4), m0=4)
mus = np.array(rb.lhs_sample(spec.p, B, spec.bounds, seed=3))
ctx = rb.mg_context_for(prob, mus)
g = torch.Generator(device="cuda").manual_seed(1)
L = rb.padded_len(n, B)
mask = torch.zeros(B, n, n, n, dtype=torch.float64, device="cuda"); mask[:, 1:, 1:, 1:] = 1
x = torch.zeros(L, dtype=torch.float64, device="cuda"); x[:B * n ** 3] = torch.randn(B * n ** 3, generator=g, device="cuda", dtype=torch.float64) * mask.view(-1)
r = torch.zeros_like(x); r[:B * n ** 3] = torch.randn(B * n ** 3, generator=g, device="cuda", dtype=torch.float64) * mask.view(-1)
out = {}
for mode in range(3):
    y = torch.zeros_like(x)
    f = lambda: _native.call("rbws_level_kernel", ctx.handle, prob.finest_level, mode, x.data_ptr(), r.data_ptr(), y.data_ptr(), 0)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nb = (16 if mode == 0 else 24) + 112 * spec.n_terms / B
    out[mode] = (ms, nb * (n - 1) ** 3 * B / ms / 1e6, y[: B * n ** 3].cpu().numpy())
if args.child:
    np.save("/tmp/fem_child.npy", np.stack([out[m][2] for m in range(3)]))
    print(" ".join(f"{out[m][0]:.4f}:{out[m][1]:.0f}" for m in range(3)))
    sys.exit(0)
env = dict(os.environ, RBWS_FEM_ZM="0")
old = subprocess.run([sys.executable, __file__, "--n", str(n), "--batch", str(B), "--child"], env=env, capture_output=True, text=True).stdout.split()
ref = np.load("/tmp/fem_child.npy")
for m in range(3):
    d = np.abs(out[m][2] - ref[m]).max() / np.abs(ref[m]).max()
    print(f"mode {m}: zmarch {out[m][0]:.4f} ms ({out[m][1]:.0f} GB/s) | old {old[m]} | max rel diff {d:.2e}")
