"""Multi-GPU plumbing for parameter-batch sharding (one process per GPU).

Parameter instances are independent, so a batch is split across ranks with no
collective on the data path.  The only communication is
host-side bookkeeping: gathering iteration counts / residuals for reporting
and the max-over-ranks timing reduction.  bench.py's rank flow (``rank_shard``,
the timed region, the reports) goes through these helpers, and
tests/test_bench_ranks_gloo.py runs that flow with two gloo ranks on CPU.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of `count` items owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_parameters(mus, rank: int, world: int) -> np.ndarray:
    mus = np.atleast_2d(np.asarray(mus, dtype=np.float64))
    lo, hi = shard_bounds(len(mus), rank, world)
    return mus[lo:hi]


def gather_reports(reports, group=None) -> list:
    """All ranks' SolveReports in global parameter order (torch.distributed, any backend)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return list(reports)
    world = dist.get_world_size(group)
    payload = [(r.iterations, float(r.true_residual), bool(r.converged), list(r.history))
               for r in reports]
    out = [None] * world
    dist.all_gather_object(out, payload, group=group)
    merged = []
    for part in out:
        merged.extend(part)
    return merged


def gather_values(value, group=None) -> list:
    """Every rank's (small, picklable) value in rank order; [value] without a process group."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return [value]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, value, group=group)
    return out


def max_over_ranks(value: float, device=None) -> float:
    """Maximum of a per-rank scalar (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
