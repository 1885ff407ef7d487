"""rbi-msrbcg at the configs[1] grid (64^3 thermal 2x2x1): train, then time one batched solve
(live CUDA events); run under ncu for the projection kernels' DRAM throughput.

    python tools/msrb_profile.py [--batch 64] [--N 8] [--K 4]
"""
import argparse, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_13862_b200 as rb

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--N", type=int, default=8)
ap.add_argument("--K", type=int, default=4)
args = ap.parse_args()
spec = rb.thermal_block((2, 2, 1))
prob = rb.ParametricProblem(spec, levels=5, m0=4)
train = rb.sample_mus(spec, 64, seed=1000)
hf = rb.HighFidelitySolver(prob, delta=1e-14, l_max=100)
t0 = time.perf_counter()
hier = rb.msrb_train(train, args.N, args.K, hf, prob)
torch.cuda.synchronize()
print(f"train {time.perf_counter() - t0:.2f}s")
test = rb.sample_mus(spec, args.batch, seed=2000)
x, reps = rb.rbi_msrbcg_solve(prob, test, hier, delta=1e-10, l_max=60)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
x, reps = rb.rbi_msrbcg_solve(prob, test, hier, delta=1e-10, l_max=60)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"rbi-msrbcg batch {args.batch}: {ms:.1f} ms ({args.batch / ms * 1e3:.1f} solves/s), "
      f"mean iterations {np.mean(reps.iterations):.2f}, converged {bool(np.all(reps.converged))}")
