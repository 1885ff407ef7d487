"""Slab-decomposed MGCG for one large instance (BASELINE configs[4]).

The reference solves a single parameter with ``mgcg_solve`` (multigrid.py:225-232
-> krylov.py:42-109) on one CPU process.  ``SlabSolver`` runs the same
preconditioned CG with the V-cycle of multigrid.py:205-222 on a grid cut into
``nslabs`` slabs of whole z-planes (C ABI ``rbws_slab_*``):

* one process, ``nslabs`` slabs on its GPU (halo planes exchanged by device
  copies) — used to check the decomposition against the oracle on one GPU;
* one process per GPU under ``torch.distributed`` (``group`` given): each rank
  holds ``nslabs / world`` consecutive slabs and exchanges halo planes and
  dot-product partials with NCCL over NVLink.

Slabs never assemble the full solution: ``load``/``store`` move the owned
planes of a padded single-instance vector (``x`` or the rhs ``f``).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native
from .grid import ParametricProblem, padded_len
from .krylov import OperatorError, SolveReport

JACOBI_OMEGA = 0.7
MIN_SLAB_PLANES = 8  # slab.cu kMinSlabPlanes


def slab_partition(cells, nslabs: int):
    """Host mirror of slab_create's decomposition (slab.cu): the first distributed
    level and, per distributed level, the owned planes [k0, k1) of every slab."""
    cells = list(cells)
    L = len(cells)
    n = cells[-1]
    if nslabs < 1 or n % (2 * nslabs) or n // nslabs < 4:
        raise ValueError("finest grid needs an even number >= 4 of planes per slab")
    ld = L - 1
    while ld - 1 >= 1 and cells[ld - 1] % nslabs == 0 and cells[ld - 1] // nslabs >= MIN_SLAB_PLANES:
        ld -= 1
    own = {l: [(r * cells[l] // nslabs, (r + 1) * cells[l] // nslabs) for r in range(nslabs)]
           for l in range(ld, L)}
    return ld, own


class SlabSolver:
    """One parameter instance of ``problem`` solved on z-slabs.

    ``nslabs``: slabs in the whole job (default: world size, or 1).
    ``group``: a ``torch.distributed`` process group for one-process-per-GPU runs
    (the NCCL unique id is broadcast over it); None = every slab in this process.
    """

    def __init__(self, problem: ParametricProblem, nslabs: int | None = None, group=None,
                 omega: float = JACOBI_OMEGA, transport: str = "auto"):
        _native.require_cuda()
        self.problem = problem
        nprocs, prank = 1, 0
        nid = None
        if group is not None:
            import torch.distributed as dist
            nprocs, prank = dist.get_world_size(group), dist.get_rank(group)
        if nslabs is None:
            nslabs = nprocs
        if nslabs % nprocs:
            raise ValueError("slabs must divide evenly over the processes")
        self.nslabs, self.nprocs, self.rank = int(nslabs), nprocs, prank
        self.nlocal = self.nslabs // nprocs
        self.ld, self.own = slab_partition(problem.cells, self.nslabs)
        if transport not in ("auto", "copy", "nccl"):
            raise ValueError(f"unknown transport {transport!r}")
        if nprocs > 1 and transport == "copy":
            raise ValueError("slabs on several processes exchange through NCCL")
        if nprocs == 1 and transport == "nccl":  # loopback: NCCL send/recv between own slabs
            buf = (ctypes.c_uint8 * 128)()
            _native.call("rbws_comm_unique_id", buf)
            nid = buf
        self.transport = "nccl" if (nprocs > 1 or transport == "nccl") else "copy"
        if nprocs > 1:
            import torch.distributed as dist
            buf = (ctypes.c_uint8 * 128)()
            if prank == 0:
                _native.call("rbws_comm_unique_id", buf)
            obj = [bytes(buf) if prank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0), group=group)
            buf = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
            nid = buf
        s = ctypes.c_void_p()
        _native.call("rbws_slab_create", ctypes.byref(s), problem.handle, self.nslabs,
                     self.nlocal, nid, nprocs, prank, float(omega))
        self._s = s
        self.mu = None
        n = problem.n
        first = prank * self.nlocal
        self.planes = (self.own[problem.levels - 1][first][0],
                       self.own[problem.levels - 1][first + self.nlocal - 1][1])

    def __del__(self):
        s = getattr(self, "_s", None)
        if s is not None and s.value and _native._lib is not None:
            _native._lib.rbws_slab_destroy(s)

    def setup(self, mu, stream=None):
        """mg_context_for (multigrid.py:191-202) for one parameter."""
        import torch
        mu = self.problem.spec.check_mus(mu)
        if len(mu) != 1:
            raise ValueError("the slab solver takes one parameter")
        self.mu = mu[0]
        self.theta = torch.as_tensor(self.problem.spec.thetas(mu)[0], dtype=torch.float64,
                                     device="cuda").contiguous()
        bad = ctypes.c_int(0)
        _native.call("rbws_slab_setup", self._s, self.theta.data_ptr(), ctypes.byref(bad),
                     _native.stream_ptr(stream))
        if bad.value:
            raise OperatorError("coarsest operator not SPD for this parameter")
        return self

    def load(self, which: str, v, p0: int = 0, stream=None):
        """Copy global planes [p0, p0 + planes) of the padded single-instance tensor
        ``v`` (device or pinned host) into the owned planes of ``x`` or ``f``."""
        n = self.problem.n
        planes = v.numel() // (n * n)
        _native.call("rbws_slab_load", self._s, 1 if which == "f" else 0, v.data_ptr(), int(p0),
                     int(min(planes, n - p0)), _native.stream_ptr(stream))

    def store(self, v, p0: int = 0, stream=None):
        """Owned planes of the solution into the padded tensor ``v`` (planes from p0)."""
        n = self.problem.n
        planes = v.numel() // (n * n)
        _native.call("rbws_slab_store", self._s, 0, v.data_ptr(), int(p0),
                     int(min(planes, n - p0)), _native.stream_ptr(stream))

    def prolong_x(self, ec, stream=None):
        """x = P ec: warm start from a full coarse solution (n/2 cells, one instance)."""
        n = self.problem.n
        if ec.numel() < padded_len(n // 2, 1) - 2 * (n // 2) ** 2:
            raise ValueError("coarse vector does not match n/2 cells")
        _native.call("rbws_slab_prolong_x", self._s, ec.data_ptr(), _native.stream_ptr(stream))

    def solve(self, delta: float = 1e-10, l_max: int = 60, stream=None) -> SolveReport:
        """PCG with the V-cycle preconditioner from the loaded x (krylov.py:42-109)."""
        if delta <= 0:
            raise ValueError("tolerance must be positive")
        if l_max < 0:
            raise ValueError("l_max must be non-negative")
        it = ctypes.c_int(0)
        st = ctypes.c_int(0)
        tr = ctypes.c_double(0.0)
        hist = np.zeros(l_max + 1)
        t0 = time.perf_counter()
        _native.call("rbws_slab_solve", self._s, float(delta), int(l_max), ctypes.byref(it),
                     hist.ctypes.data, ctypes.byref(tr), ctypes.byref(st),
                     _native.stream_ptr(stream))
        wall = time.perf_counter() - t0
        if st.value & 1:
            raise OperatorError("non-positive curvature; operator not SPD")
        k = it.value
        return SolveReport(
            method="mgcg", iterations=k, history=[float(v) for v in hist[:k + 1]],
            converged=bool(tr.value <= delta), true_residual=float(tr.value), wall_time=wall,
            delta=delta, l_max=l_max, mu=None if self.mu is None else np.asarray(self.mu),
            absolute_norms=bool(st.value & 4),
            config={"slabs": self.nslabs, "processes": self.nprocs, "smoother": "jacobi",
                    "transport": self.transport,
                    "nu": 1, "first_distributed_level": self.ld})


def slab_mgcg_solve(problem: ParametricProblem, mu, f=None, x0=None, nslabs: int = 1,
                    delta: float = 1e-10, l_max: int = 60, solver: SlabSolver | None = None,
                    transport: str = "auto"):
    """Single-process convenience: full padded f / x0 in, full padded x out."""
    import torch
    s = solver or SlabSolver(problem, nslabs=nslabs, transport=transport)
    s.setup(mu)
    n = problem.n
    f = problem.rhs() if f is None else f
    s.load("f", f)
    if x0 is None:
        x0 = torch.zeros(padded_len(n, 1), dtype=torch.float64, device="cuda")
    s.load("x", x0)
    rep = s.solve(delta=delta, l_max=l_max)
    x = torch.zeros(padded_len(n, 1), dtype=torch.float64, device="cuda")
    s.store(x)
    return x, rep
