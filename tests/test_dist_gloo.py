"""World-size-2 gloo test of the parameter-sharding host logic (CPU only)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_13862_b200 import dist as rd
    from paper_2311_13862_b200.krylov import SolveReport
    from paper_2311_13862_b200.problems import sample_mus, thermal_block
    mus = sample_mus(thermal_block((2, 2, 1)), 7, seed=3)
    mine = rd.shard_parameters(mus, rank, world)
    # stand-in per-instance results: iterations = global index
    lo, hi = rd.shard_bounds(len(mus), rank, world)
    reps = [SolveReport("mgcg", g, [1.0] * (g + 1), True, 1e-11, 0.0, 1e-10, 40) for g in range(lo, hi)]
    merged = rd.gather_reports(reps)
    t = rd.max_over_ranks(10.0 + rank)
    q.put((rank, mine.tolist(), [m[0] for m in merged], t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover_exactly():
    from paper_2311_13862_b200.dist import shard_bounds
    for count in (0, 1, 7, 1024):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(count, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    from paper_2311_13862_b200.problems import sample_mus, thermal_block
    mus = sample_mus(thermal_block((2, 2, 1)), 7, seed=3)
    got = np.concatenate([np.asarray(r[1]) for r in res])
    np.testing.assert_array_equal(got, mus)
    for r in res:
        assert r[2] == list(range(7))   # gathered in global order on every rank
        assert r[3] == 11.0             # max over ranks
