"""World-size-2 gloo model of the multi-process slab path (CPU only).

Each rank holds one z-slab of every distributed level exactly as slab.cu lays it
out (owned planes [k0, k1) plus one halo plane on each side) and performs the
same communication the native solver issues through NCCL: halo planes sent
to / received from the neighbouring ranks (XCHG_UP: top owned plane -> lower
halo of the rank above; XCHG_DOWN: bottom owned plane -> upper halo of the rank
below), the all-gather of each rank's coarse planes into the first replicated
level (chunk = the rank's planes at offset rank * chunk, as the in-place
ncclAllGather), and the all-gather of dot-product partials.  The oracle's
operators then show that these halos are exactly what the stencils, the
restriction and the dots need: slab-local results equal the global ones.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(buf, n, nz, rank, world, dirs):
    """slab.cu Slab::xchg between processes; buf: (nz + 2, n, n) planes k0-1 .. k1."""
    import torch.distributed as dist
    ops = []
    if rank + 1 < world:
        if dirs & 1:
            ops.append(dist.P2POp(dist.isend, buf[nz].contiguous(), rank + 1))
        if dirs & 2:
            top = torch.empty(n, n, dtype=buf.dtype)
            ops.append(dist.P2POp(dist.irecv, top, rank + 1))
    if rank > 0:
        if dirs & 1:
            bot = torch.empty(n, n, dtype=buf.dtype)
            ops.append(dist.P2POp(dist.irecv, bot, rank - 1))
        if dirs & 2:
            ops.append(dist.P2POp(dist.isend, buf[1].contiguous(), rank - 1))
    for w in dist.batch_isend_irecv(ops) if ops else []:
        w.wait()
    if rank + 1 < world and dirs & 2:
        buf[nz + 1] = top
    if rank > 0 and dirs & 1:
        buf[0] = bot


def _embed(buf, k0, n):
    """Slab planes k0-1 .. k1 into a zero global padded vector (n^3)."""
    full = np.zeros((n, n, n))
    for t in range(buf.shape[0]):
        k = k0 - 1 + t
        if 0 <= k < n:
            full[k] = buf[t].numpy()
    return full.ravel()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import problems as op
        from paper_2311_13862_b200.slab import slab_partition
        n, m0 = 32, 4
        ospec = op.thermal_block((2, 2, 2))
        oprob = op.OracleProblem(ospec, n, m0)
        mu = op.sample_mus(ospec, 1, seed=4)[0]
        cells = oprob.cells
        L = len(cells)
        ld, own = slab_partition(cells, world)
        out = {"ld": ld}
        rng = np.random.default_rng(0)
        for l in range(ld, L):
            nl = cells[l]
            k0, k1 = own[l][rank]
            nz = k1 - k0
            x = op.interior_to_padded(rng.standard_normal((nl - 1) ** 3), nl).reshape(nl, nl, nl)
            buf = torch.zeros(nz + 2, nl, nl, dtype=torch.float64)
            buf[1:nz + 1] = torch.from_numpy(x[k0:k1].copy())
            _exchange(buf, nl, nz, rank, world, 3)
            lo_ok = np.array_equal(buf[0].numpy(), x[k0 - 1] if k0 >= 1 else np.zeros((nl, nl)))
            hi_ok = np.array_equal(buf[nz + 1].numpy(), x[k1] if k1 < nl else np.zeros((nl, nl)))
            # stencil on the owned planes from the slab alone == global stencil
            A = oprob.operator(mu, level=l)
            y_slab = op.interior_to_padded(A @ op.padded_to_interior(_embed(buf, k0, nl), nl), nl)
            y_glob = op.interior_to_padded(A @ op.padded_to_interior(x.ravel(), nl), nl)
            sl = slice(max(1, k0) * nl * nl, k1 * nl * nl)
            op_err = float(np.max(np.abs(y_slab[sl] - y_glob[sl])))
            # restriction of the owned coarse planes after the upward exchange only
            nc = nl // 2
            P = oprob.prolongations[l - 1]
            up = torch.zeros_like(buf)
            up[1:nz + 1] = buf[1:nz + 1]
            _exchange(up, nl, nz, rank, world, 1)
            rc_slab = op.interior_to_padded(P.T @ op.padded_to_interior(_embed(up, k0, nl), nl), nc)
            rc_glob = op.interior_to_padded(P.T @ op.padded_to_interior(x.ravel(), nl), nc)
            K0, K1 = k0 // 2, k1 // 2
            csl = slice(max(1, K0) * nc * nc, K1 * nc * nc)
            r_err = float(np.max(np.abs(rc_slab[csl] - rc_glob[csl])))
            gath_err = None
            if l == ld:  # into the first replicated level: all-gather of the owned planes
                chunk = (nc // world) * nc * nc
                mine = torch.from_numpy(rc_slab[K0 * nc * nc:K1 * nc * nc].copy())
                parts = [torch.empty(chunk, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, mine)
                full = torch.cat(parts).numpy()
                gath_err = float(np.max(np.abs(full - rc_glob)))
            # dot partials: all-gathered, summed in rank order
            part = torch.tensor([float((x[k0:k1] ** 2).sum())], dtype=torch.float64)
            parts = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, part)
            dot_err = abs(float(sum(p.item() for p in parts)) - float((x ** 2).sum()))
            out[l] = (lo_ok, hi_ok, op_err, r_err, gath_err, dot_err)
        q.put((rank, out))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_slab_partition_rules():
    from paper_2311_13862_b200.slab import slab_partition
    cells = (4, 8, 16, 32, 64, 128, 256, 512)
    for R, want_ld in ((1, 1), (2, 2), (4, 3), (8, 4)):
        ld, own = slab_partition(cells, R)
        assert ld == want_ld
        for l, spans in own.items():
            assert spans[0][0] == 0 and spans[-1][1] == cells[l]
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all((b - a) % 2 == 0 for a, b in spans)   # even: restriction ownership
    with pytest.raises(ValueError):
        slab_partition((4, 8, 16), 8)   # 2 planes per slab
    with pytest.raises(ValueError):
        slab_partition((4, 8, 16, 32), 3)


def test_gloo_world2_slab_halos_restriction_dots():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, out in res.items():
        assert out["ld"] == 2            # 32 and 16 cells distributed, 8 and 4 replicated
        for l in (2, 3):
            lo_ok, hi_ok, op_err, r_err, gath_err, dot_err = out[l]
            assert lo_ok and hi_ok, (rank, l)
            assert op_err <= 1e-12, (rank, l, op_err)
            assert r_err <= 1e-12, (rank, l, r_err)
            assert dot_err <= 1e-9
        assert out[2][4] is not None and out[2][4] <= 1e-12
