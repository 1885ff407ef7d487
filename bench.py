"""Benchmark: warm-started (RBI-)MGCG solves/s to 1e-10 on the BASELINE workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C]

One step = the online stage for one batch of test parameters, resident in
HBM: batched mg_context_for (per-mu coarse operators + coarsest Cholesky),
the batched L1ROC online solve (affine reduced assembly + least squares +
warm-start expansion) and the batched MGCG refinement to the tolerance —
the reference's t_on protocol (experiment.py:31-33) for a whole batch.
Offline greedy training runs once before timing.  Multi-GPU: one process
per GPU, parameters sharded by rank (weak scaling, no data-path collective).

--impl reference times the CPU restatement of the reference algorithm
(oracle/, the reference package is Python and cannot travel to the box) on
all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "warm-started MGCG solves/s to 1e-10 rel. residual; stencil HBM GB/s vs peak"

# BASELINE.json configs (index = position in "configs")
CONFIGS = {
    0: dict(workload="thermal-block 2x1x1, 32^3 cells, r=10 from 256 train, batch 64, tol 1e-10",
            kind="tb", blocks=(2, 1, 1), n=32, m0=4, r=10, n_train=256, batch=64, delta=1e-10,
            degenerate="stop"),
    1: dict(workload="thermal-block 2x2x1, 64^3 cells, r=20 from 1024 train, batch 1024, tol 1e-10",
            kind="tb", blocks=(2, 2, 1), n=64, m0=4, r=20, n_train=1024, batch=1024, delta=1e-10,
            e2e_sizes=[1024]),
    2: dict(workload="thermal-block 2x2x2, 128^3 cells, r=30 from 4096 train, batch 512, tol 1e-12",
            kind="tb", blocks=(2, 2, 2), n=128, m0=4, r=30, n_train=4096, batch=512, delta=1e-12,
            scaling="strong", degenerate="stop"),
    3: dict(workload="smooth affine (6 modes), 256^3 cells, r=40 from 2048 train, batch 128, tol 1e-12",
            kind="smooth", blocks=None, n=256, m0=4, r=40, n_train=2048, batch=128, delta=1e-12,
            chunk=64, e2e_sub=32, degenerate="stop"),
    4: dict(workload="thermal-block 2x2x2, 512^3 cells, one instance slab-decomposed along z "
                     "(one slab per GPU); RB warm start r=30 from 4096 train at 128^3, prolonged; "
                     "tol 1e-10",
            kind="tb", blocks=(2, 2, 2), n=512, m0=4, r=30, n_train=4096, rb_n=128, batch=1,
            delta=1e-10, slab=True),
}
L_MAX = 60

# algorithmic bytes per interior node and instance for each profiled kernel class
CLASS_NAMES = ["fine_p_update_apply_dot", "fine_cg_update", "fine_pre_residual", "fine_restrict",
               "fine_prolong", "fine_prolong_post_smooth", "fine_p_update", "coarse_levels",
               "scalars"]
# reads + writes per interior node and instance:
#  p-update+apply: s, p_old -> p_new | cg: p, x, r -> x, r | pre: b, dinv -> r1
#  restrict: r1 -> bc, uc (2/8) + dinv_c (1/8) | prolong+post (fused): b, dinv, e (1/8) -> s
CLASS_BYTES = {0: 24.0, 1: 40.0, 2: 24.0, 3: 11.0, 4: 25.0, 5: 25.0, 6: 24.0}
# fused pre-smoothing (b, dinv -> t, the x/z-restricted residual: 1/4) and its y pass
# (t 1/4 -> bc, uc 2/8, dinv_c 1/8)
FUSED_PRE_BYTES = 18.0
FUSED_RESTRICT_Y_BYTES = 5.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def make_spec(cfg, pkg):
    if cfg["kind"] == "tb":
        return pkg.thermal_block(cfg["blocks"])
    return pkg.smooth_affine(6)


def make_ospec(cfg):
    from oracle import problems as op
    if cfg["kind"] == "tb":
        return op.thermal_block(cfg["blocks"])
    return op.smooth_affine(6)


# ---------------------------------------------------------------- b200 arm

def _traffic(kernel, bytes_per_launch, cfg):
    """DRAM bytes per launch for the dominant kernel from the committed ncu capture
    (profiles/r02_traffic.json, configs[1]); scaled to this run's average launch by the
    captured traffic/algorithmic ratio. None for workloads that were not captured."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic.json")
    if cfg["workload"] != CONFIGS[1]["workload"] or not os.path.exists(path):
        return None, None
    with open(path) as fh:
        cap = json.load(fh)
    if kernel not in cap:
        return None, None
    ratio = cap[kernel]["dram_bytes"] / cap[kernel]["algorithmic_bytes"]
    return int(ratio * bytes_per_launch), f"{cap['source']}; dram/algorithmic = {ratio:.3f}"


def rank_shard(args, cfg, rank, world, sampler):
    """This rank's test parameters.  weak: every rank solves its own batch of the config's
    size (seed 2000 + rank), whole-job units = world x batch; strong: one global batch
    (seed 2000) split into contiguous shards (dist.shard_parameters), units = the batch."""
    from paper_2311_13862_b200 import dist as rdist
    batch = args.batch or cfg["batch"]
    scaling = args.scaling or cfg.get("scaling", "weak")
    if scaling == "strong":
        mus = rdist.shard_parameters(sampler(batch, 2000), rank, world)
        lo, hi = rdist.shard_bounds(batch, rank, world)
        return {"mus": mus, "local": len(mus), "total": batch, "scaling": "strong",
                "desc": f"global batch {batch} sharded: rank {rank} of {world} owns [{lo}, {hi})"}
    return {"mus": sampler(batch, 2000 + rank), "local": batch, "total": world * batch,
            "scaling": "weak", "desc": f"{batch} parameters per rank (seed 2000 + rank)"}


def run_b200(args, rank, world, dist):
    import torch

    import build as _build
    if rank == 0:
        _build.build(verbose=False)
    if dist is not None:
        dist.barrier()
    import paper_2311_13862_b200 as rb
    from paper_2311_13862_b200 import _native
    from paper_2311_13862_b200 import dist as rdist

    cfg = CONFIGS[args.config]
    n, m0 = cfg["n"], cfg["m0"]
    delta = cfg["delta"]
    spec = make_spec(cfg, rb)
    levels = rb.problems.levels_for(n, m0)
    prob = rb.ParametricProblem(spec, levels=levels, m0=m0)
    train = rb.sample_mus(spec, cfg["n_train"], seed=1000)
    shard = rank_shard(args, cfg, rank, world, lambda c, s: rb.sample_mus(spec, c, seed=s))
    test, batch = shard["mus"], shard["local"]

    t0 = time.perf_counter()
    hf = rb.HighFidelitySolver(prob, delta=1e-14, l_max=100)
    # the reference raises on a snapshot numerically inside the basis (rb.py:116-117); the
    # configs whose greedy reaches that (degenerate="stop") end it there instead, flagged as
    # saturated in the model (configs[1] keeps the reference behaviour)
    model = rb.l1roc_offline(train, cfg["r"], hf, prob, seed=0,
                             on_degenerate=cfg.get("degenerate", "raise"))
    torch.cuda.synchronize()
    t_off = time.perf_counter() - t0
    log(f"[rank {rank}] offline greedy: N={model.dim} saturated={model.saturated} "
        f"in {t_off:.2f}s")

    # instances per device-resident sub-batch (bounded by HBM for the largest grids)
    chunk = min(batch, args.chunk or cfg.get("chunk", batch))
    chunks = [test[c:c + chunk] for c in range(0, batch, chunk)]
    ctx = rb.MgContext(prob, chunk)
    f = prob.rhs()
    method = rb.MethodConfig("rbi-mgcg", delta=delta, l_max=L_MAX, N=model.dim)
    xbuf = torch.empty(rb.padded_len(n, chunk), dtype=torch.float64, device="cuda")
    state = {}

    def step():
        reps = []
        for part in chunks:
            rb.mg_context_for(prob, part, ctx=ctx)
            x, r = rb.rbi_pcg_solve(rb.BatchOperator(ctx), f, method, mg_ctx=ctx,
                                    l1roc_model=model, x0_out=xbuf)
            reps.append(r)   # lazy report batches: no per-instance host work in the step
        state["reps"], state["x"] = reps, x
        return x

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # zero-initialised MGCG on the same batch for reference (outside the timed region)
    _, zreps = rb.mgcg_solve(None, f, None, ctx, delta=delta, l_max=L_MAX)  # last sub-batch
    zero_iters = float(np.mean([r.iterations for r in zreps]))

    # ---- timed region (device-resident inputs; the default device-side graph PCG loop,
    # no per-kernel events)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    lc0 = _native.launch_count()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        torch.cuda.nvtx.range_push("rbws_timed")   # ncu --nvtx-include rbws_timed/
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    launches = _native.launch_count() - lc0
    ms = ev0.elapsed_time(ev1)
    ms_max = rdist.max_over_ranks(ms, device="cuda")
    ms_step = ms_max / args.steps
    value = shard["total"] * args.steps / (ms_max / 1e3)
    reps = [r for batch_reps in state["reps"] for r in batch_reps]
    all_reps = rdist.gather_reports(reps)            # every rank's reports, global order
    iters = [r[0] if isinstance(r, tuple) else r.iterations for r in all_reps]
    worst_res = max(r[1] if isinstance(r, tuple) else r.true_residual for r in all_reps)
    converged = all(r[2] if isinstance(r, tuple) else r.converged for r in all_reps)
    my_iters = [r.iterations for r in reps]

    # ---- per-kernel-class breakdown (roofline): the same K steps once more with the CUDA
    # event profiler on (host-driven PCG loop, an event pair per kernel class); not the
    # timed region above, whose number it does not touch
    torch.cuda.synchronize()
    _native.call("rbws_batch_profile", ctx.handle, 1)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(args.steps):
        step()
    pe1.record(stream)
    torch.cuda.synchronize()
    ms_prof = pe0.elapsed_time(pe1)
    NC = len(CLASS_NAMES)
    pms = np.zeros(NC)
    pcalls = np.zeros(NC, dtype=np.int64)
    punits = np.zeros(NC, dtype=np.int64)
    _native.call("rbws_batch_profile_read", ctx.handle, pms.ctypes.data, pcalls.ctypes.data,
                 punits.ctypes.data, NC)
    _native.call("rbws_batch_profile", ctx.handle, 0)

    # ---- end to end through the public API with host buffers: host mu in, solutions
    # out to pinned host memory, sub-batches pipelined (paper_2311_13862_b200.pipeline)
    del state["x"]
    scw = bool(_native.load().rbws_batch_stored_weights(ctx.handle))
    fused = bool(_native.load().rbws_batch_fused_restrict(ctx.handle))
    pre_sw = bool(_native.load().rbws_batch_pre_scaled(ctx.handle))
    cg_fused = bool(_native.load().rbws_batch_cg_fused(ctx.handle))
    del ctx, xbuf
    torch.cuda.empty_cache()
    e2e_sub = min(batch, args.e2e_sub or cfg.get("e2e_sub", 512))
    sizes = [int(v) for v in args.e2e_sizes.split(",")] if args.e2e_sizes else \
        (cfg.get("e2e_sizes") if batch == cfg["batch"] else None)
    pipe = rb.HostPipeline(prob, method, model, sub_batch=e2e_sub,
                           tail=args.e2e_tail or None, sizes=sizes)
    hbuf = torch.empty(batch * n ** 3, dtype=torch.float64, pin_memory=True)
    mus_host = np.ascontiguousarray(test)
    pipe.solve(mus_host, hbuf)  # warm-up (untimed)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        # back-to-back calls: a call's last downloads overlap the next call's solves;
        # every download is inside the timed region (the caller waits for them below)
        reps_e = pipe.solve(mus_host, hbuf, sync=False)
    stream.wait_stream(pipe.copy_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = rdist.max_over_ranks(e0.elapsed_time(e1), device="cuda")
    e2e_value = shard["total"] * args.steps / (e2e_ms / 1e3)
    e2e_iters_ok = all(a.iterations == b for a, b in zip(reps_e, my_iters))
    tb = shard["total"]  # whole job: every rank's copies
    h2d = tb * spec.n_terms * 8
    d2h = tb * n ** 3 * 8 + tb * (L_MAX + 1) * 8 + tb * (4 + 8 + 4)

    # ---- roofline of the dominant fine-level kernel class
    peak, peak_kind = peaks()
    nodes = (n - 1) ** 3
    # stored face weights (SCW kernels): +24 B/node in every finest-level stencil sweep
    class_bytes = {k: v + (24.0 if (scw and k != 3) else 0.0) for k, v in CLASS_BYTES.items()}
    if fused:  # pre-smoothing + x/z restriction in one kernel: r1 never written
        class_bytes[2] = FUSED_PRE_BYTES + (24.0 if scw else 0.0)
        class_bytes[3] = FUSED_RESTRICT_Y_BYTES
    # scaled-weights pre-smoothing kernels: the 1/diag vector is not streamed (-8 B/node); the
    # bytes of the operation as the reference states it (b, D^-1 in) are reported next to it
    op_bytes = dict(class_bytes)
    if pre_sw:
        class_bytes[2] -= 8.0
    # CG update fused with the next V-cycle's pre-smoothing residual + x/z restriction
    # (p, x, r -> x, r, t 1/4): the pre-smoothing class then only holds each solve's first V-cycle
    if cg_fused:
        class_bytes[1] = 42.0 + (24.0 if scw else 0.0)
        op_bytes[1] = 42.0 + (24.0 if scw else 0.0)
    table = {}
    for k in range(NC):
        if pcalls[k] == 0:
            continue
        row = {"ms_total": round(float(pms[k]), 3), "launches": int(pcalls[k]),
               "ms_per_launch": round(float(pms[k]) / pcalls[k], 4),
               "share": round(float(pms[k]) / ms_prof, 4)}
        if k in class_bytes:
            gbs = class_bytes[k] * nodes * punits[k] / (pms[k] / 1e3) / 1e9
            row["achieved_gbs"] = round(gbs, 1)
            row["bytes_per_node"] = class_bytes[k]
            if op_bytes[k] != class_bytes[k]:
                row["op_bytes_per_node"] = op_bytes[k]
                row["op_gbs"] = round(gbs * op_bytes[k] / class_bytes[k], 1)
        elif CLASS_NAMES[k] == "coarse_levels":
            # algorithmic bytes of one V-cycle's coarse levels per instance: 76 B per node
            # of every smoothed coarse level (pre-smoothing residual 24, restriction 11,
            # prolongation 17, post-smoothing 24) + the coarsest Cholesky solve
            m0 = prob.cells[0]
            cb = sum(76.0 * (c - 1) ** 3 for c in prob.cells[1:-1]) + \
                8.0 * ((m0 - 1) ** 6 + 2 * (m0 - 1) ** 3)
            row["achieved_gbs"] = round(cb * punits[k] / (pms[k] / 1e3) / 1e9, 1)
            row["bytes_per_instance"] = cb
        table[CLASS_NAMES[k]] = row
    ran = [k for k in class_bytes if pcalls[k]]
    if ran:
        dom = max(ran, key=lambda k: pms[k])
        dom_bytes = class_bytes[dom] * nodes * punits[dom] / pcalls[dom]
        dom_s = pms[dom] / pcalls[dom] / 1e3
        achieved = dom_bytes / dom_s / 1e9
        traffic, tsrc = _traffic(CLASS_NAMES[dom], dom_bytes, cfg)
        roofline = {"bound": "hbm", "kernel": CLASS_NAMES[dom], "achieved": round(achieved, 1),
                    "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                    "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_kind,
                    "bytes_per_launch": int(dom_bytes),
                    "bytes_per_node": class_bytes[dom], "stored_weights": scw,
                    "fused_pre_restrict": fused, "scaled_weights_pre": pre_sw,
                    "cg_update_fused_with_pre_smoothing": cg_fused}
    else:  # the warm start already met the tolerance: no PCG iteration ran
        roofline = {"bound": "hbm", "kernel": None, "achieved": None, "peak": peak,
                    "unit": "GB/s", "frac": None, "traffic": None, "peak_source": peak_kind}

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, model, test, my_iters, budget_s=args.cpu_budget)
    fracs = rdist.gather_values(roofline.get("frac"))

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": shard["scaling"], "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded log-uniform parameters; no dataset)",
        "config": {"workload": cfg["workload"], "batch_per_gpu": batch,
                   "global_batch": shard["total"], "sharding": shard["desc"], "sub_batch": chunk,
                   "grid_cells": n,
                   "levels": levels, "rb_dim": model.dim, "n_train": cfg["n_train"],
                   "tolerance": delta, "smoother": "jacobi(0.7), nu=1",
                   "parallelism": f"parameter-sharded x{world}",
                   "l2": "inputs larger than L2 (working set >> 126 MB)",
                   "mean_iterations_warm": round(float(np.mean(iters)), 3),
                   "max_iterations_warm": int(max(iters)),
                   "mean_iterations_zero_init": round(zero_iters, 3),
                   "all_converged": converged, "max_true_residual": worst_res,
                   "t_offline_s": round(t_off, 3)},
        "e2e": {"value": round(e2e_value, 2), "unit": "solves/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "sub_batches": pipe.schedule(batch),
                "api": "HostPipeline.solve (host mu -> pinned host solutions)",
                "iterations_match_device_run": bool(e2e_iters_ok)},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "roofline_pass": ("per-class CUDA events over a second run of the same K steps "
                          "(host-driven PCG loop); the timed region runs the device-side "
                          f"graph loop: {ms_prof / args.steps:.3f} ms/step profiled vs "
                          f"{ms / args.steps:.3f} timed on rank {rank}"),
        "roofline_frac_per_rank": fracs,
        "kernels": table,
        "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)


def slab_bytes_per_node(cells, iters):
    """Algorithmic HBM bytes of one slab solve per finest-level node (DESIGN.md §3 table):
    per PCG iteration the finest level moves 124 B/node and a coarse level l
    76 B per level-l node (pre 24 + restriction 11 + prolongation 17 + post-smoothing 24);
    once per solve: ||f|| (8), two residuals (2 x 24), the first V-cycle."""
    nf = (cells[-1] - 1) ** 3
    coarse = sum(76.0 * (c - 1) ** 3 for c in cells[1:-1]) / nf
    vcyc = 24 + 11 + 25 + coarse
    return iters * (124.0 + coarse) + 8 + 48 + vcyc


def run_slab(args, rank, world, dist):
    """configs[4]: one 512^3 instance per step, slab-decomposed over the GPUs (strong scaling)."""
    import torch

    import build as _build
    if rank == 0:
        _build.build(verbose=False)
    if dist is not None:
        dist.barrier()
    import paper_2311_13862_b200 as rb
    from paper_2311_13862_b200 import _native

    cfg = CONFIGS[args.config]
    n, m0, nc = cfg["n"], cfg["m0"], cfg["rb_n"]
    delta = cfg["delta"]
    spec = make_spec(cfg, rb)
    prob = rb.ParametricProblem(spec, levels=rb.problems.levels_for(n, m0), m0=m0)
    cprob = rb.ParametricProblem(spec, levels=rb.problems.levels_for(nc, m0), m0=m0)
    train = rb.sample_mus(spec, cfg["n_train"], seed=1000)
    t0 = time.perf_counter()
    hf = rb.HighFidelitySolver(cprob, delta=1e-14, l_max=100)
    model = rb.l1roc_offline(train, cfg["r"], hf, cprob, seed=0, on_degenerate="stop")
    torch.cuda.synchronize()
    t_off = time.perf_counter() - t0
    log(f"[rank {rank}] offline greedy at {nc}^3: N={model.dim} in {t_off:.2f}s")

    group = dist.group.WORLD if dist is not None else None
    nslabs = world * max(1, args.slabs_per_gpu)
    solver = rb.SlabSolver(prob, nslabs=nslabs, group=group)
    f = prob.rhs()
    solver.load("f", f)
    k0, k1 = solver.planes
    mus = rb.sample_mus(spec, args.warmup + args.steps + 1, seed=3000)   # same on every rank
    cctx = rb.MgContext(cprob, 1)
    fc = cprob.rhs()
    lifts = []  # warm start prolonged nc -> 2nc -> ... -> n/2 (full vectors, every rank)
    c = nc
    while c < n // 2:
        lifts.append(torch.zeros(rb.padded_len(2 * c, 1), dtype=torch.float64, device="cuda"))
        c *= 2
    stream = torch.cuda.current_stream()

    stored = torch.cuda.Event()  # e2e: the previous solution's download (x reusable after)

    def warm_start(mu):
        rb.mg_context_for(cprob, mu[None], ctx=cctx)
        u, _ = rb.l1roc_online(model, rb.BatchOperator(cctx), fc)
        c = nc
        for buf in lifts:
            buf.zero_()
            _native.call("rbws_prolong_add", 2 * c, 1, u.data_ptr(), buf.data_ptr(),
                         _native.stream_ptr())
            u, c = buf, 2 * c
        torch.cuda.current_stream().wait_event(stored)
        solver.prolong_x(u)

    def step(mu):
        solver.setup(mu[None])
        warm_start(mu)
        return solver.solve(delta=delta, l_max=L_MAX)

    for w in range(args.warmup):
        step(mus[w])
    # zero-initialised solve of the first timed parameter (outside the timed region)
    solver.setup(mus[args.warmup][None])
    solver.load("x", torch.zeros(rb.padded_len(n, 1), dtype=torch.float64, device="cuda"))
    zero_rep = solver.solve(delta=delta, l_max=L_MAX)
    torch.cuda.synchronize()

    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    lc0 = _native.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    with ClockSampler(torch.cuda.current_device()) as clocks:
        torch.cuda.nvtx.range_push("rbws_timed")
        ev0.record(stream)
        for s_ in range(args.steps):
            reps.append(step(mus[args.warmup + s_]))
        ev1.record(stream)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    launches = _native.launch_count() - lc0
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = args.steps / (ms_max / 1e3)
    iters = [r.iterations for r in reps]

    # ---- end to end: host parameter in, this rank's planes of the solution out to pinned
    # host memory, every step
    hbuf = torch.empty((k1 - k0) * n * n, dtype=torch.float64, pin_memory=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    copy = torch.cuda.Stream()
    e0.record(stream)
    for s_ in range(args.steps):
        step(np.asarray(mus[args.warmup + s_]))
        # download this rank's planes on a side stream; the next step's setup and warm
        # start overlap it and only the overwrite of x (prolong_x) waits for it
        copy.wait_stream(stream)
        solver.store(hbuf, p0=k0, stream=copy)
        stored.record(copy)
    stream.wait_stream(copy)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = args.steps / (float(e2e_ms.item()) / 1e3)

    peak, peak_kind = peaks()
    bpn = slab_bytes_per_node(prob.cells, float(np.mean(iters)))
    achieved = bpn * (n - 1) ** 3 / (ms_max / args.steps / 1e3) / 1e9 / world
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded log-uniform parameters; no dataset)",
        "config": {"workload": cfg["workload"], "grid_cells": n, "levels": prob.levels,
                   "slabs": nslabs, "planes_per_slab": n // nslabs,
                   "first_distributed_level": solver.ld, "transport": solver.transport,
                   "rb_dim": model.dim, "rb_grid_cells": nc, "n_train": cfg["n_train"],
                   "tolerance": delta, "smoother": "jacobi(0.7), nu=1",
                   "parallelism": f"z-slabs x{nslabs} over {world} GPU(s)",
                   "l2": "inputs larger than L2 (1 GB per vector)",
                   "iterations_warm": iters, "iterations_zero_init": zero_rep.iterations,
                   "all_converged": all(r.converged for r in reps),
                   "max_true_residual": max(r.true_residual for r in reps),
                   "t_offline_s": round(t_off, 3)},
        "e2e": {"value": round(e2e_value, 4), "unit": "solves/s",
                "h2d_bytes_per_step": spec.n_terms * 8,
                "d2h_bytes_per_step": (k1 - k0) * n * n * 8,
                "api": "SlabSolver.setup/prolong_x/solve/store (host mu -> pinned host planes)"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "whole slab solve (all levels, per GPU)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None,
                     "peak_source": peak_kind, "bytes_per_fine_node": round(bpn, 1),
                     "note": "algorithmic bytes of the whole step / step time (setup, warm "
                             "start, halo exchanges included)"},
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = slab_cpu_baseline(cfg, iters, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)


def slab_cpu_baseline(cfg, gpu_iters, budget_s=15.0):
    """The oracle MGCG (single core) cannot hold a 512^3 operator in seconds: time its
    per-iteration cost at 64^3 and scale by DoFs to the GPU's iteration count."""
    _single_thread_blas()
    from oracle import problems as op
    from oracle import solvers as so
    ospec = make_ospec(cfg)
    ns = 64
    oprob = op.OracleProblem(ospec, ns, cfg["m0"])
    mu = op.sample_mus(ospec, 1, seed=3000)[0]
    A, f = oprob.operator(mu), oprob.rhs()
    ctx = so.mg_context_for(oprob, mu)
    t0 = time.perf_counter()
    done = 0
    per_it = []
    while time.perf_counter() - t0 < budget_s:
        t1 = time.perf_counter()
        _, rep = so.mgcg_solve(A, f, np.zeros_like(f), ctx, delta=cfg["delta"], l_max=L_MAX)
        per_it.append((time.perf_counter() - t1) / max(rep.iterations, 1))
        done += 1
    scale = ((cfg["n"] - 1) / (ns - 1)) ** 3
    t_solve = float(np.median(per_it)) * scale * float(np.mean(gpu_iters))
    return {"value": round(1.0 / t_solve, 6), "unit": "solves/s", "cores": 1, "kind": "port",
            "sample": f"{done} zero-init oracle MGCG solves at {ns}^3 (per-iteration time, "
                      f"single-threaded), scaled by DoFs x{scale:.0f} to 512^3 at the GPU's "
                      f"mean iteration count; extrapolated, not measured at 512^3"}


def cpu_baseline(cfg, model, test, gpu_iters, budget_s=15.0):
    """Oracle RBI-MGCG per parameter (single core) on a bounded sample."""
    _single_thread_blas()
    from oracle import problems as op
    from oracle import solvers as so
    ospec = make_ospec(cfg)
    t0 = time.perf_counter()
    oprob = op.OracleProblem(ospec, cfg["n"], cfg["m0"])
    t_build = time.perf_counter() - t0
    omodel = so.OracleL1rocModel(model.basis_numpy(), model.transform, model.collocation,
                                 model.solution_points, model.residual_points,
                                 np.asarray(model.chosen if model.chosen is not None else []),
                                 model.indicator_history, model.saturated)
    done, match, t_solve = 0, 0, 0.0
    for m, mu in enumerate(test):
        t1 = time.perf_counter()
        _, rep = so.rbi_mgcg_solve(oprob, mu, omodel, delta=cfg["delta"], l_max=L_MAX)
        t_solve += time.perf_counter() - t1
        done += 1
        match += int(abs(rep.iterations - gpu_iters[m]) <= 1)
        if t_solve > budget_s:
            break
    return {"value": round(done / t_solve, 4), "unit": "solves/s", "cores": 1, "kind": "port",
            "sample": f"{done} of the step's test parameters, oracle RBI-MGCG (mg_context_for + "
                      f"l1roc_online + MGCG to tol) single-threaded; operator assembly "
                      f"{t_build:.1f}s excluded; iteration counts within +-1 of the GPU: "
                      f"{match}/{done}"}


# ---------------------------------------------------------------- assembled (FEM) problems

FEM_WORKLOAD = ("example-1 (the reference's own Q1 FEM problem: oscillatory coefficient, "
                "mu-dependent Dirichlet data), {n}^3 cells, m0=4, r={r} from {t} LHS train, "
                "batch {b}, tol 1e-10")


def run_fem(args, rank, world, dist):
    """`--problem example-1`: RBI-MGCG on the reference's own assembled problem (stored
    27-point coefficients on every level).  Step = mg_context_for + L1ROC warm start + MGCG
    for the batch with the right-hand sides already assembled (the reference's t_on
    protocol excludes operator and rhs assembly, experiment.py:31-33)."""
    import torch

    import build as _build
    if rank == 0:
        _build.build(verbose=False)
    if dist is not None:
        dist.barrier()
    import paper_2311_13862_b200 as rb
    from paper_2311_13862_b200 import _native

    n, m0, r, n_train = args.fem_n, 4, args.fem_r, args.fem_train
    batch = args.batch or 256
    delta = 1e-10
    spec = rb.get_problem(args.problem)
    levels = rb.problems.levels_for(n, m0)
    t0 = time.perf_counter()
    prob = rb.ParametricProblem(spec, levels=levels, m0=m0)
    t_setup = time.perf_counter() - t0
    train = np.array(rb.problems.lhs_sample(spec.p, n_train, spec.bounds, seed=1000))
    test = np.array(rb.problems.lhs_sample(spec.p, batch, spec.bounds, seed=2000 + rank))
    t0 = time.perf_counter()
    model = rb.l1roc_offline(train, r, rb.HighFidelitySolver(prob, delta=1e-14, l_max=100),
                             prob, seed=0, on_degenerate="stop")
    torch.cuda.synchronize()
    t_off = time.perf_counter() - t0
    F = prob.rhs(test)
    ctx = rb.MgContext(prob, batch)
    method = rb.MethodConfig("rbi-mgcg", delta=delta, l_max=L_MAX, N=model.dim)
    xbuf = torch.empty(rb.padded_len(n, batch), dtype=torch.float64, device="cuda")
    state = {}

    def step(f):
        rb.mg_context_for(prob, test, ctx=ctx)
        x, reps = rb.rbi_pcg_solve(rb.BatchOperator(ctx), f, method, mg_ctx=ctx,
                                   l1roc_model=model, x0_out=xbuf)
        state["reps"] = reps
        return x

    for _ in range(args.warmup):
        step(F)
    torch.cuda.synchronize()
    _, zreps = rb.mgcg_solve(None, F, None, ctx, delta=delta, l_max=L_MAX)
    zero_iters = float(np.mean([z.iterations for z in zreps]))
    stream = torch.cuda.current_stream()
    lc0 = _native.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step(F)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = _native.launch_count() - lc0
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * batch * args.steps / (ms_max / 1e3)
    reps = state["reps"]
    iters = [q.iterations for q in reps]

    # e2e: rhs batch from pinned host memory, solutions back to pinned host memory
    fh = F.cpu().pin_memory()
    xh = torch.empty(batch * n ** 3, dtype=torch.float64, pin_memory=True)
    fd = torch.empty_like(F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        fd.copy_(fh, non_blocking=True)
        x = step(fd)
        xh.copy_(x[: batch * n ** 3], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * batch * args.steps / (float(e2e_ms.item()) / 1e3)

    # roofline: the finest-level stored 27-point apply over the batch, timed alone
    peak, peak_kind = peaks()
    A = rb.BatchOperator(ctx)
    xv = torch.randn(rb.padded_len(n, batch), dtype=torch.float64, device="cuda")
    A.apply(xv)
    reps_k = 20
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(reps_k):
        A.apply(xv)
    k1.record(stream)
    torch.cuda.synchronize()
    k_ms = k0.elapsed_time(k1) / reps_k
    bpn = float(prob.apply_bytes_per_node(ctx))
    kbytes = bpn * (n - 1) ** 3 * batch
    achieved = kbytes / (k_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "stored27_apply (finest level, batch)",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_kind,
                "bytes_per_launch": int(kbytes), "bytes_per_node": bpn,
                "ms_per_launch": round(k_ms, 4)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = fem_cpu_baseline(spec, n, m0, model, test, iters, budget_s=args.cpu_budget)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded LHS parameters, sampling.py:8-27; no dataset)",
        "config": {"workload": FEM_WORKLOAD.format(n=n, r=r, t=n_train, b=batch),
                   "batch_per_gpu": batch, "grid_cells": n, "levels": levels,
                   "rb_dim": model.dim, "n_train": n_train, "tolerance": delta,
                   "smoother": "jacobi(0.7), nu=1", "parallelism": f"parameter-sharded x{world}",
                   "mean_iterations_warm": round(float(np.mean(iters)), 3),
                   "max_iterations_warm": int(max(iters)),
                   "mean_iterations_zero_init": round(zero_iters, 3),
                   "all_converged": all(q.converged for q in reps),
                   "t_setup_s": round(t_setup, 2), "t_offline_s": round(t_off, 2),
                   "l2": "inputs larger than L2"},
        "e2e": {"value": round(e2e_value, 2), "unit": "solves/s",
                "h2d_bytes_per_step": int(F.numel() * 8),
                "d2h_bytes_per_step": int(batch * n ** 3 * 8),
                "api": "assembled rhs (pinned host) -> rbi_pcg_solve -> pinned host solutions"},
        "gpu_launches": int(launches), "roofline": roofline, "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)


def _fem2_desc(args):
    if args.fem2_method == "mgcg":
        return "zero-init MGCG"
    return f"RBI-MGCG (L1ROC r={args.fem_r} from {args.fem_train} LHS training parameters)"


FEM2_METRIC = {
    "rbi-mgcg": "warm-started MGCG solves/s to 1e-10 rel. residual (example-2, plane-Jacobi)",
    "mgcg": "zero-init MGCG solves/s to 1e-10 rel. residual (example-2, plane-Jacobi)"}
FEM2_WORKLOAD = ("example-2 (the reference's mixed problem: zero-flux face x=1, anisotropic "
                 "quadrant coefficient, mu-dependent source), {n}^3 cells, m0=4, {m} "
                 "with the plane-Jacobi smoother (reference default), batch {b}, tol 1e-10")


def run_fem2(args, rank, world, dist):
    """`--problem example-2`: HighFidelitySolver(method="mgcg") semantics (hf.py:40-57) on
    the reference's example-2 in the full-node layout (csrc/planes.cu).  Step =
    mg_context_for (theta-combined coefficients, banded Cholesky of every z-plane block and
    of the coarsest level) + zero-init MGCG to 1e-10 for the batch, right-hand sides
    resident (assembly excluded, experiment.py:31-33)."""
    import torch

    import build as _build
    if rank == 0:
        _build.build(verbose=False)
    if dist is not None:
        dist.barrier()
    import paper_2311_13862_b200 as rb
    from paper_2311_13862_b200 import _native, fem
    from paper_2311_13862_b200.fem_fn import FnFemProblem, _ptr, mg_context_for, mgcg_solve
    from paper_2311_13862_b200.problems import levels_for, lhs_sample

    n, m0 = args.fem_n, 4
    batch = args.batch or 64
    delta = 1e-10
    spec = fem.example2()
    levels = levels_for(n, m0)
    t0 = time.perf_counter()
    prob = FnFemProblem(spec, levels=levels, m0=m0)
    t_setup = time.perf_counter() - t0
    test = np.array(lhs_sample(spec.p, batch, spec.bounds, seed=2000 + rank))
    F = prob.rhs(test)
    state = {}
    rbi = args.fem2_method == "rbi-mgcg"
    model, t_off = None, 0.0
    if rbi:  # the reference's rbi-mgcg on Ex.2: L1ROC greedy from an LHS training set
        train = np.array(lhs_sample(spec.p, args.fem_train, spec.bounds, seed=1000))
        t0 = time.perf_counter()
        hf = rb.HighFidelitySolver(prob, delta=1e-14, l_max=100)
        model = rb.l1roc_offline(train, args.fem_r, hf, prob, seed=0, on_degenerate="stop")
        torch.cuda.synchronize()
        t_off = time.perf_counter() - t0
        log(f"[rank {rank}] example-2 greedy: N={model.dim} in {t_off:.2f}s")
    cfg = rb.MethodConfig(args.fem2_method, delta=delta, l_max=L_MAX,
                          N=model.dim if model is not None else 0)

    def step(f):
        ctx = mg_context_for(prob, test)
        x, reps = rb.rbi_pcg_solve(rb.BatchOperator(ctx), f, cfg, mg_ctx=ctx,
                                   l1roc_model=model)
        state["reps"], state["ctx"] = reps, ctx
        return x

    for _ in range(args.warmup):
        step(F)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    lc0 = _native.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step(F)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = _native.launch_count() - lc0
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * batch * args.steps / (ms_max / 1e3)
    reps = state["reps"]
    iters = [int(i) for i in reps.iterations]
    _, zreps = mgcg_solve(state["ctx"], F, delta=delta, l_max=L_MAX)  # untimed reference
    zero_iters = float(np.mean(zreps.iterations))

    # e2e: rhs batch from pinned host memory, free-DoF solutions back to pinned host memory
    fh = F.cpu().pin_memory()
    xh = torch.empty_like(fh).pin_memory()
    fd = torch.empty_like(F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        fd.copy_(fh, non_blocking=True)
        x = step(fd)
        xh.copy_(x, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * batch * args.steps / (float(e2e_ms.item()) / 1e3)

    # roofline: the finest-level plane-block solve (16 lanes per plane system), timed alone;
    # algorithmic bytes = the band factors (M (w+1) doubles per plane) read by BOTH the
    # forward and the backward substitution (a 2.3 MB factor per plane does not stay on
    # chip between the passes) + r read/write/read-back + x read/write
    peak, peak_kind = peaks()
    ctx = state["ctx"]
    c = n
    M, w = (c + 1) ** 2, c + 2
    nsys = batch * (c + 1)
    kbytes = 2 * nsys * M * (w + 1) * 8 + 5 * batch * (c + 1) ** 3 * 8
    r = torch.randn(batch, (c + 1) ** 3, dtype=torch.float64, device="cuda")
    xk = torch.zeros_like(r)
    st = _native.stream_ptr()

    def solve_once():
        _native.call("rbws_fn_band_solve", batch, c, 1, _ptr(ctx.bands[-1]), _ptr(r), _ptr(xk),
                     0.6, 1, st)

    solve_once()
    reps_k = 10
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(reps_k):
        solve_once()
    k1.record(stream)
    torch.cuda.synchronize()
    k_ms = k0.elapsed_time(k1) / reps_k
    achieved = kbytes / (k_ms / 1e3) / 1e9
    # DRAM bytes of one such launch from the ncu --set full capture (64^3, 64 instances)
    traffic = 19_569_175_000 + 241_493_248 if (n, batch) == (64, 64) else None
    roofline = {"bound": "hbm", "kernel": "band_solve_sub_kernel (finest z-plane blocks, batch)",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": "profiles/r01i_example2.md (ncu --set full, one finest sweep, "
                                  "64^3 x 64; dram/algorithmic = 1.01)",
                "peak_source": peak_kind,
                "bytes_per_launch": int(kbytes), "ms_per_launch": round(k_ms, 4)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = fem2_cpu_baseline(n, m0, test, iters, budget_s=args.cpu_budget, model=model)
    line = {
        "metric": FEM2_METRIC[args.fem2_method],
        "value": round(value, 2), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded LHS parameters, sampling.py:8-27; no dataset)",
        "config": {"workload": FEM2_WORKLOAD.format(n=n, b=batch, m=_fem2_desc(args)),
                   "batch_per_gpu": batch, "grid_cells": n, "levels": levels,
                   "tolerance": delta, "smoother": "plane-jacobi(0.6), nu=1",
                   "layout": "full-node (c+1)^3 per instance", "parallelism": f"parameter-sharded x{world}",
                   "method": args.fem2_method,
                   "rb_dim": model.dim if model is not None else 0,
                   "n_train": args.fem_train if rbi else 0, "t_offline_s": round(t_off, 2),
                   "mean_iterations": round(float(np.mean(iters)), 3), "max_iterations": int(max(iters)),
                   "mean_iterations_zero_init": round(zero_iters, 3),
                   "all_converged": bool(np.all(reps.converged)),
                   "t_setup_s": round(t_setup, 2), "l2": "inputs larger than L2"},
        "e2e": {"value": round(e2e_value, 2), "unit": "solves/s",
                "h2d_bytes_per_step": int(F.numel() * 8), "d2h_bytes_per_step": int(F.numel() * 8),
                "api": "assembled rhs (pinned host) -> rbi_pcg_solve (full-node batch) -> "
                       "pinned host solutions"},
        "gpu_launches": int(launches), "roofline": roofline, "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)


def fem2_cpu_baseline(n, m0, test, gpu_iters, budget_s=15.0, model=None):
    """Oracle MGCG (plane-Jacobi, splu plane factors as the reference; with ``model`` the
    L1ROC warm start on the GPU-trained model first) on example-2, single core, on a bounded
    sample of the batch's parameters."""
    from oracle import fem as of
    from oracle import solvers as so
    from paper_2311_13862_b200.problems import levels_for
    t0 = time.perf_counter()
    op = of.OracleFemProblem(of.Example2(), levels=levels_for(n, m0), m0=m0)
    t_asm = time.perf_counter() - t0
    omodel = None if model is None else so.OracleL1rocModel(
        model.basis_numpy(), model.transform, model.collocation, model.solution_points,
        model.residual_points, np.asarray(model.chosen if model.chosen is not None else []),
        model.indicator_history, model.saturated)
    done, agree, t_solve = 0, 0, 0.0
    for i, mu in enumerate(test):
        t1 = time.perf_counter()
        _, rep = so.rbi_mgcg_solve(op, mu, omodel, delta=1e-10, l_max=L_MAX, smoother="auto")
        t_solve += time.perf_counter() - t1
        done += 1
        agree += int(abs(rep.iterations - gpu_iters[i]) <= (1 if omodel is not None else 0))
        if t_solve > budget_s:
            break
    return {"value": round(done / t_solve, 4), "unit": "solves/s", "cores": 1, "kind": "port",
            "sample": f"{done} of the step's parameters, oracle "
                      f"{'RBI-MGCG (L1ROC warm start on the GPU-trained model) ' if omodel is not None else 'MGCG '}"
                      f"(operator + rhs + mg_context_for incl. splu plane factors + MGCG) "
                      f"single-threaded; assembly {t_asm:.1f}s excluded; iteration counts "
                      f"agreeing with the GPU: {agree}/{done}"}


def fem_cpu_baseline(spec, n, m0, model, test, gpu_iters, budget_s=15.0):
    """Oracle RBI-MGCG on example-1 (single core) on a bounded sample."""
    _single_thread_blas()
    from oracle import fem as of
    from oracle import solvers as so
    t0 = time.perf_counter()
    oprob = of.OracleFemProblem(of.Example1(), levels=int(np.log2(n // m0)) + 1, m0=m0)
    t_build = time.perf_counter() - t0
    omodel = so.OracleL1rocModel(model.basis_numpy(), model.transform, model.collocation,
                                 model.solution_points, model.residual_points,
                                 np.asarray(model.chosen if model.chosen is not None else []),
                                 model.indicator_history, model.saturated)
    done, match, t_solve = 0, 0, 0.0
    for m, mu in enumerate(test):
        t1 = time.perf_counter()
        _, rep = so.rbi_mgcg_solve(oprob, mu, omodel, delta=1e-10, l_max=L_MAX)
        t_solve += time.perf_counter() - t1
        done += 1
        match += int(abs(rep.iterations - gpu_iters[m]) <= 1)
        if t_solve > budget_s:
            break
    return {"value": round(done / t_solve, 4), "unit": "solves/s", "cores": 1, "kind": "port",
            "sample": f"{done} of the step's test parameters, oracle RBI-MGCG single-threaded; "
                      f"assembly {t_build:.1f}s excluded; iterations within +-1 of the GPU: "
                      f"{match}/{done}"}


# ---------------------------------------------------------------- reference arm

_W = {}


def _single_thread_blas():
    """One BLAS/OpenMP thread per process (the pool supplies the parallelism)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _ref_worker_init(cfg, model_state):
    _single_thread_blas()
    from oracle import problems as op
    from oracle import solvers as so
    _W["oprob"] = op.OracleProblem(make_ospec(cfg), cfg["n"], cfg["m0"])
    _W["model"] = so.OracleL1rocModel(*model_state)
    _W["cfg"] = cfg


def _ref_solve(mu):
    from oracle import solvers as so
    _, rep = so.rbi_mgcg_solve(_W["oprob"], mu, _W["model"], delta=_W["cfg"]["delta"],
                               l_max=L_MAX)
    return rep.iterations


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.problem:
        return run_reference_fem(args, world)
    if CONFIGS[args.config].get("slab"):
        return run_reference_slab(args, world)
    import multiprocessing as mp
    from oracle import problems as op
    from oracle import solvers as so
    cfg = CONFIGS[args.config]
    ospec = make_ospec(cfg)
    n, m0 = cfg["n"], cfg["m0"]
    cores = os.cpu_count() or 1
    oprob = op.OracleProblem(ospec, n, m0)
    train = op.sample_mus(ospec, cfg["n_train"], seed=1000)
    test = op.sample_mus(ospec, args.batch or cfg["batch"], seed=2000)

    def hf(mu):  # reference HighFidelitySolver(method="mgcg") (hf.py:40-57)
        A, f = oprob.operator(mu), oprob.rhs()
        x, _ = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(oprob, mu), 1e-14, 100)
        return x

    t0 = time.perf_counter()
    model = so.l1roc_offline(list(train), cfg["r"], hf, oprob.operator, oprob.operator_rows,
                             oprob.rhs, seed=0, on_degenerate=cfg.get("degenerate", "raise"))
    t_off = time.perf_counter() - t0
    log(f"[reference] offline greedy N={model.dim} in {t_off:.1f}s")
    state = (model.basis, model.transform, model.collocation, model.solution_points,
             model.residual_points, model.chosen, model.indicator_history, model.saturated)
    sample = cores * max(1, args.ref_per_core)
    ctxm = mp.get_context("fork")
    with ctxm.Pool(cores, initializer=_ref_worker_init, initargs=(cfg, state)) as pool:
        k = 0
        for _ in range(args.warmup):
            pool.map(_ref_solve, [test[(k + i) % len(test)] for i in range(cores)])
            k += cores
        t1 = time.perf_counter()
        iters = []
        for _ in range(args.steps):
            iters += pool.map(_ref_solve, [test[(k + i) % len(test)] for i in range(sample)])
            k += sample
        el = time.perf_counter() - t1
    value = args.steps * sample / el
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded log-uniform parameters; no dataset)", "impl": "reference",
        "config": {"workload": cfg["workload"], "rb_dim": model.dim,
                   "mean_iterations_warm": round(float(np.mean(iters)), 3),
                   "t_offline_s": round(t_off, 1)},
        "cpu_baseline": {"value": round(value, 4), "unit": "solves/s", "cores": cores,
                         "kind": "port",
                         "sample": f"{sample} test parameters per step ({args.ref_per_core} per "
                                   f"core), oracle restatement of the reference RBI-MGCG "
                                   f"(scipy.sparse), process pool over all host cores"},
        "e2e": {"value": round(value, 4), "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _ref_fem_init(n, m0, model_state):
    _single_thread_blas()
    from oracle import fem as of
    from oracle import solvers as so
    _W["oprob"] = of.OracleFemProblem(of.Example1(), levels=int(np.log2(n // m0)) + 1, m0=m0)
    _W["model"] = so.OracleL1rocModel(*model_state)


def _ref_fem_solve(mu):
    from oracle import solvers as so
    _, rep = so.rbi_mgcg_solve(_W["oprob"], mu, _W["model"], delta=1e-10, l_max=L_MAX)
    return rep.iterations


def _ref_fem2_init(n, m0, model_state=None):
    _single_thread_blas()
    from oracle import fem as of
    from oracle import solvers as so
    _W["oprob"] = of.OracleFemProblem(of.Example2(), levels=int(np.log2(n // m0)) + 1, m0=m0)
    _W["model"] = None if model_state is None else so.OracleL1rocModel(*model_state)


def _ref_fem2_solve(mu):
    from oracle import solvers as so
    _, rep = so.rbi_mgcg_solve(_W["oprob"], mu, _W["model"], delta=1e-10, l_max=L_MAX,
                               smoother="auto")
    return rep.iterations


def run_reference_fem2(args, world):
    """`--impl reference --problem example-2`: the oracle restatement of the reference's
    zero-init plane-Jacobi MGCG (mg_context_for incl. splu plane factors + MGCG per
    parameter, as HighFidelitySolver(method="mgcg")), process pool over all host cores."""
    import multiprocessing as mp
    from oracle import fem as of
    from oracle import solvers as so
    n, m0 = args.fem_n, 4
    spec = of.Example2()
    test = np.array(so.lhs_sample(spec.p, args.batch or 64, spec.bounds, seed=2000))
    cores = os.cpu_count() or 1
    sample = cores * max(1, args.ref_per_core)
    state, t_off = None, 0.0
    if args.fem2_method == "rbi-mgcg":  # the oracle greedy (HighFidelitySolver "mgcg")
        oprob = of.OracleFemProblem(spec, levels=int(np.log2(n // m0)) + 1, m0=m0)
        train = np.array(so.lhs_sample(spec.p, args.fem_train, spec.bounds, seed=1000))

        def hf(mu):
            A, f = oprob.operator(mu), oprob.rhs(mu)
            x, _ = so.mgcg_solve(A, f, np.zeros_like(f),
                                 so.mg_context_for(oprob, mu, smoother="auto"), 1e-14, 100)
            return x

        t0 = time.perf_counter()
        model = so.l1roc_offline(list(train), args.fem_r, hf, oprob.operator,
                                 oprob.operator_rows, oprob.rhs, seed=0, on_degenerate="stop")
        t_off = time.perf_counter() - t0
        state = (model.basis, model.transform, model.collocation, model.solution_points,
                 model.residual_points, model.chosen, model.indicator_history, model.saturated)
    with mp.get_context("fork").Pool(cores, initializer=_ref_fem2_init,
                                     initargs=(n, m0, state)) as pool:
        k = 0
        for _ in range(args.warmup):
            pool.map(_ref_fem2_solve, [test[(k + i) % len(test)] for i in range(cores)])
            k += cores
        t1 = time.perf_counter()
        iters = []
        for _ in range(args.steps):
            iters += pool.map(_ref_fem2_solve, [test[(k + i) % len(test)] for i in range(sample)])
            k += sample
        el = time.perf_counter() - t1
    value = args.steps * sample / el
    line = {
        "metric": FEM2_METRIC[args.fem2_method],
        "value": round(value, 4), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded LHS parameters, sampling.py:8-27; no dataset)",
        "impl": "reference",
        "config": {"workload": FEM2_WORKLOAD.format(n=n, b=args.batch or 64, m=_fem2_desc(args)),
                   "method": args.fem2_method, "t_offline_s": round(t_off, 1),
                   "mean_iterations": round(float(np.mean(iters)), 3)},
        "cpu_baseline": {"value": round(value, 4), "unit": "solves/s", "cores": cores,
                         "kind": "port",
                         "sample": f"{sample} test parameters per step ({args.ref_per_core} per "
                                   f"core), oracle restatement of the reference "
                                   f"{args.fem2_method} with the plane-Jacobi smoother on "
                                   f"example-2 (scipy.sparse, splu plane factors), process "
                                   f"pool over all host cores"},
        "e2e": {"value": round(value, 4), "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_fem(args, world):
    """`--impl reference --problem example-1`: the oracle restatement of the reference's
    RBI-MGCG on its own FEM problem, process pool over all host cores (rank 0 only)."""
    import multiprocessing as mp
    from oracle import fem as of
    from oracle import solvers as so
    if args.problem == "example-2":
        return run_reference_fem2(args, world)
    if args.problem != "example-1":
        raise SystemExit(f"no reference arm for problem {args.problem!r}")
    n, m0 = args.fem_n, 4
    spec = of.Example1()
    oprob = of.OracleFemProblem(spec, levels=int(np.log2(n // m0)) + 1, m0=m0)
    train = np.array(so.lhs_sample(spec.p, args.fem_train, spec.bounds, seed=1000))
    test = np.array(so.lhs_sample(spec.p, args.batch or 256, spec.bounds, seed=2000))

    def hf(mu):  # HighFidelitySolver(method="mgcg") semantics (hf.py:40-57)
        A, f = oprob.operator(mu), oprob.rhs(mu)
        x, _ = so.mgcg_solve(A, f, np.zeros_like(f), so.mg_context_for(oprob, mu), 1e-14, 100)
        return x

    t0 = time.perf_counter()
    model = so.l1roc_offline(list(train), args.fem_r, hf, oprob.operator, oprob.operator_rows,
                             oprob.rhs, seed=0, on_degenerate="stop")
    t_off = time.perf_counter() - t0
    state = (model.basis, model.transform, model.collocation, model.solution_points,
             model.residual_points, model.chosen, model.indicator_history, model.saturated)
    cores = os.cpu_count() or 1
    sample = cores * max(1, args.ref_per_core)
    with mp.get_context("fork").Pool(cores, initializer=_ref_fem_init,
                                     initargs=(n, m0, state)) as pool:
        k = 0
        for _ in range(args.warmup):
            pool.map(_ref_fem_solve, [test[(k + i) % len(test)] for i in range(cores)])
            k += cores
        t1 = time.perf_counter()
        iters = []
        for _ in range(args.steps):
            iters += pool.map(_ref_fem_solve, [test[(k + i) % len(test)] for i in range(sample)])
            k += sample
        el = time.perf_counter() - t1
    value = args.steps * sample / el
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded LHS parameters, sampling.py:8-27; no dataset)",
        "impl": "reference",
        "config": {"workload": FEM_WORKLOAD.format(n=n, r=args.fem_r, t=args.fem_train,
                                                   b=args.batch or 256),
                   "rb_dim": model.dim, "mean_iterations_warm": round(float(np.mean(iters)), 3),
                   "t_offline_s": round(t_off, 1)},
        "cpu_baseline": {"value": round(value, 4), "unit": "solves/s", "cores": cores,
                         "kind": "port",
                         "sample": f"{sample} test parameters per step ({args.ref_per_core} per "
                                   f"core), oracle restatement of the reference RBI-MGCG on "
                                   f"example-1 (scipy.sparse), process pool over all host cores"},
        "e2e": {"value": round(value, 4), "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_slab(args, world):
    """configs[4] on the CPU: the oracle cannot assemble a 512^3 operator within a bounded
    sample, so each step times zero-init oracle MGCG solves at 64^3 and scales the time per
    iteration by the DoF ratio at the 64^3 iteration count (stated in cpu_baseline.sample)."""
    _single_thread_blas()
    from oracle import problems as op
    from oracle import solvers as so
    cfg = CONFIGS[args.config]
    ospec = make_ospec(cfg)
    ns = 64
    oprob = op.OracleProblem(ospec, ns, cfg["m0"])
    mus = op.sample_mus(ospec, args.warmup + args.steps, seed=3000)
    scale = ((cfg["n"] - 1) / (ns - 1)) ** 3
    est, iters = [], []
    for k, mu in enumerate(mus):
        A, f = oprob.operator(mu), oprob.rhs()
        ctx = so.mg_context_for(oprob, mu)
        t0 = time.perf_counter()
        _, rep = so.mgcg_solve(A, f, np.zeros_like(f), ctx, delta=cfg["delta"], l_max=L_MAX)
        el = time.perf_counter() - t0
        if k >= args.warmup:
            est.append(el * scale)
            iters.append(rep.iterations)
    value = len(est) / sum(est)
    line = {
        "metric": METRIC, "value": round(value, 6), "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sum(est) / len(est) * 1e3, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded log-uniform parameters; no dataset)", "impl": "reference",
        "config": {"workload": cfg["workload"], "mean_iterations_64": float(np.mean(iters))},
        "cpu_baseline": {"value": round(value, 6), "unit": "solves/s", "cores": 1, "kind": "port",
                         "sample": f"one zero-init oracle MGCG solve at {ns}^3 per step "
                                   f"(single-threaded), time scaled by the DoF ratio x{scale:.0f} "
                                   f"to 512^3 at the 64^3 iteration count; extrapolated"},
        "e2e": {"value": round(value, 6), "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_dry(args, rank, world, dist):
    """--dry-run: the multi-rank flow of run_b200 (sharding, barrier-bracketed timed
    region, max over ranks, report gathering, one JSON line from rank 0) on CPU with gloo
    and a host stand-in for the solve (iterations = global parameter index), so the rank
    orchestration is testable without GPUs (tests/test_bench_ranks_gloo.py)."""
    from paper_2311_13862_b200 import dist as rdist
    from paper_2311_13862_b200.krylov import SolveReport
    from paper_2311_13862_b200.problems import sample_mus, thermal_block
    cfg = CONFIGS[args.config]
    spec = thermal_block(cfg["blocks"] or (2, 2, 1))
    shard = rank_shard(args, cfg, rank, world, lambda c, s: sample_mus(spec, c, seed=s))
    if shard["scaling"] == "strong":
        lo, _ = rdist.shard_bounds(shard["total"], rank, world)
    else:
        lo = rank * shard["local"]
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        reps = [SolveReport("rbi-mgcg", lo + i, [1.0], True, 1e-11, 0.0, 1e-10, L_MAX)
                for i in range(shard["local"])]
        time.sleep(0.01 * (1 + rank))
    ms = (time.perf_counter() - t0) * 1e3
    ms_max = rdist.max_over_ranks(ms)
    merged = rdist.gather_reports(reps)
    mus_all = rdist.gather_values(shard["mus"].tolist())
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(shard["total"] * args.steps / (ms_max / 1e3), 2),
            "unit": "solves/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": shard["scaling"], "dry_run": True,
            "config": {"workload": cfg["workload"], "global_batch": shard["total"],
                       "batch_per_gpu": shard["local"], "sharding": shard["desc"]},
            "report_order": [m[0] for m in merged],
            "mus_by_rank": mus_all}), flush=True)


def _spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: start N copies of this command as ranks
    0..N-1 (RANK/LOCAL_RANK/WORLD_SIZE, rendezvous on 127.0.0.1), the way
    torch.distributed.run would; rank 0's stdout carries the JSON line."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0, help="instances per device sub-batch")
    ap.add_argument("--e2e-sub", type=int, default=0,
                    help="instances per pipelined sub-batch of the end-to-end (host buffer) run")
    ap.add_argument("--e2e-tail", type=int, default=0,
                    help="smallest pipelined sub-batch of the end-to-end run (0: sub/4)")
    ap.add_argument("--e2e-sizes", default="",
                    help="explicit end-to-end sub-batch sizes, e.g. 512,384,128")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-per-core", type=int, default=2)
    ap.add_argument("--problem", default="",
                    help="reference problem id: example-1 (RBI-MGCG on its assembled operator) or "
                         "example-2 (zero-init plane-Jacobi MGCG, full-node layout)")
    ap.add_argument("--fem-n", type=int, default=64)
    ap.add_argument("--fem2-method", default="rbi-mgcg", choices=["rbi-mgcg", "mgcg"],
                    help="example-2: warm-started (L1ROC) or zero-init MGCG")
    ap.add_argument("--fem-r", type=int, default=10)
    ap.add_argument("--fem-train", type=int, default=256)
    ap.add_argument("--scaling", default="", choices=["", "weak", "strong"],
                    help="weak: a full batch per GPU (default); strong: one global batch "
                         "sharded by parameter across the GPUs (configs[2]'s default)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo run of the multi-rank orchestration with a stand-in solve")
    ap.add_argument("--slabs-per-gpu", type=int, default=1,
                    help="configs[4]: slabs per GPU (>1: in-process slabs exchanging by copies)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        log("note: fewer than 3 warm-up steps requested")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        sys.exit(_spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        run_reference(args, rank, max(world, args.gpus))
        return
    if args.dry_run:
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        run_dry(args, rank, world, dist)
        if dist is not None:
            dist.destroy_process_group()
        return
    import torch
    if args.gpus > 1 and torch.cuda.device_count() < world:
        raise SystemExit(f"--gpus {args.gpus}: only {torch.cuda.device_count()} CUDA devices")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.problem == "example-2":
        run_fem2(args, rank, world, dist)
    elif args.problem:
        run_fem(args, rank, world, dist)
    elif CONFIGS[args.config].get("slab"):
        run_slab(args, rank, world, dist)
    else:
        run_b200(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
