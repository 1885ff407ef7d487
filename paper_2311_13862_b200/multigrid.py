"""Batched geometric multigrid and MGCG on the B200.

B200 counterpart of reference multigrid.py:
  * ``mg_context_for`` (multigrid.py:191-202) -> per-batch native context:
    operators of every level for every mu (coarse levels as per-instance
    27-point stencils assembled from the Kronecker factors), Jacobi
    diagonals, Cholesky of the coarsest level;
  * ``mg_vcycle`` (multigrid.py:205-222) -> one V-cycle for the whole batch;
  * ``mgcg_solve`` (multigrid.py:225-232) -> native batched PCG.
The smoother is the reference's isotropic default, damped Jacobi with
omega = 0.7 (multigrid.py:26-27, 183-188).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native
from .grid import BatchOperator, ParametricProblem, padded_len
from .krylov import OperatorError, SolveReport, SolveReports

JACOBI_OMEGA = 0.7
# V-cycle smoothers (reference multigrid.py:132-152): damped Jacobi both sides, or forward
# Gauss-Seidel before / backward after the coarse correction
SMOOTHERS = ("jacobi", "gs")


class MgContext:
    """Per-batch multigrid state (reference MgContext, multigrid.py:116-129)."""

    def __init__(self, problem: ParametricProblem, capacity: int, nu: int = 1,
                 omega: float = JACOBI_OMEGA, smoother: str = "jacobi"):
        if nu < 1:
            raise ValueError("the batched V-cycle needs nu >= 1 smoothing sweeps")
        if smoother not in SMOOTHERS:
            raise ValueError(f"unknown smoother kind {smoother!r}; choices: {SMOOTHERS}")
        self.problem = problem
        self.capacity = int(capacity)
        self.nu = nu
        self.omega = omega
        self.smoother_kind = smoother
        b = ctypes.c_void_p()
        _native.call("rbws_batch_create", ctypes.byref(b), problem.handle, self.capacity, nu,
                     float(omega))
        self._b = b
        if smoother == "gs":
            _native.call("rbws_batch_set_smoother", b, 1)
        self.count = 0
        self.mus = None
        self.theta = None

    def __del__(self):
        b = getattr(self, "_b", None)
        if b is not None and b.value and _native._lib is not None:
            _native._lib.rbws_batch_destroy(b)

    @property
    def handle(self):
        return self._b

    @property
    def levels(self) -> int:
        return self.problem.levels

    def setup(self, mus, stream=None):
        """Bind the context to a batch of parameters (per-mu operators + factors)."""
        import torch
        mus = self.problem.spec.check_mus(mus)
        if len(mus) > self.capacity:
            raise ValueError(f"batch of {len(mus)} exceeds context capacity {self.capacity}")
        self.mus = mus
        self.count = len(mus)
        self.theta = torch.as_tensor(self.problem.spec.thetas(mus), dtype=torch.float64,
                                     device="cuda").contiguous()
        bad = ctypes.c_int(0)
        _native.call("rbws_batch_setup", self._b, self.theta.data_ptr(), self.count,
                     ctypes.byref(bad), _native.stream_ptr(stream))
        if bad.value:
            raise OperatorError(f"coarsest operator not SPD for {bad.value} parameter(s)")
        return self


def mg_context_for(problem: ParametricProblem, mus, nu: int = 1, smoother: str = "auto",
                   ctx: MgContext | None = None) -> MgContext:
    """Batched mg_context_for (multigrid.py:191-202).

    ``mus``: one parameter or an array (count, p).  Pass an existing ``ctx``
    to reuse its device buffers for a new batch.  Problems with free boundary nodes
    (example-2) get a full-node context (fem_fn.py; smoothers "auto" = plane-Jacobi,
    "plane-jacobi", "jacobi").
    """
    from .fem_fn import FnFemProblem
    if isinstance(problem, FnFemProblem):
        from . import fem_fn
        return fem_fn.mg_context_for(problem, mus, nu=nu, smoother=smoother)
    if smoother == "auto":  # isotropic problems: damped Jacobi (multigrid.py:183-188)
        smoother = "jacobi"
    if smoother not in SMOOTHERS:
        raise ValueError(f"smoother {smoother!r} is not on the B200 path ({SMOOTHERS})")
    mus = problem.spec.check_mus(mus)
    if (ctx is None or ctx.capacity < len(mus) or ctx.nu != nu or ctx.problem is not problem
            or ctx.smoother_kind != smoother):
        ctx = MgContext(problem, len(mus), nu=nu, smoother=smoother)
    return ctx.setup(mus)


def mg_vcycle(b, ctx: MgContext, level=None):
    """One V-cycle from zero for every instance of the batch (multigrid.py:205-222)."""
    import torch
    from .fem_fn import FnMgContext
    if isinstance(ctx, FnMgContext):
        return ctx.vcycle(b, level)
    if level is not None and level != ctx.levels - 1:
        raise ValueError("the batched V-cycle is entered on the finest level")
    n = ctx.problem.n
    if b.numel() != padded_len(n, ctx.count) and b.numel() < padded_len(n, ctx.count):
        raise ValueError("right-hand side does not match level size")
    out = torch.zeros_like(b)
    _native.call("rbws_vcycle", ctx.handle, b.data_ptr(), out.data_ptr(), _native.stream_ptr())
    return out


def mgcg_solve(A, f, x0, ctx: MgContext, delta: float = 1e-16, l_max: int = 40, mu=None,
               method: str = "mgcg", raise_on_breakdown: bool = True,
               overwrite_x0: bool = False, out_host=None, copy_stream=None):
    """Batched MGCG (multigrid.py:225-232 -> krylov.py:42-109).

    f: padded rhs, either one instance (shared) or a full batch; x0: padded
    batch of initial guesses (None = zeros), left untouched unless
    ``overwrite_x0`` (then the solve runs in x0's storage).  Returns (x, [SolveReport]).
    Full-node contexts (example-2): f / x0 are (count, (n+1)^3) full-node batches.
    """
    import torch
    from .fem_fn import FnMgContext
    if isinstance(ctx, FnMgContext):
        from . import fem_fn
        return fem_fn.mgcg_solve(ctx, f, x0, delta=delta, l_max=l_max, method=method)
    if delta <= 0:
        raise ValueError("tolerance must be positive")
    if l_max < 0:
        raise ValueError("l_max must be non-negative")
    prob = ctx.problem
    n, count = prob.n, ctx.count
    if f is None:
        f = prob.rhs(ctx.mus)
    nb = padded_len(n, count)
    if f.numel() == padded_len(n, 1) and count > 1:
        f_stride = 0
    elif f.numel() >= nb:
        f_stride = n ** 3
    else:
        raise ValueError("rhs does not match the batch")
    if x0 is None:
        x = torch.zeros(nb, dtype=torch.float64, device="cuda")
    elif overwrite_x0:
        if x0.numel() < nb or not x0.is_contiguous():
            raise ValueError("x0 does not hold the batch")
        x = x0
    else:
        x = x0.clone()
    iters = np.zeros(count, dtype=np.int32)
    hist = np.zeros((count, l_max + 1))
    tres = np.zeros(count)
    status = np.zeros(count, dtype=np.int32)
    t0 = time.perf_counter()
    if out_host is not None:
        # stream each instance's solution to pinned host memory as soon as it stops
        # iterating (copies enqueued on copy_stream)
        if not out_host.is_pinned() or out_host.numel() < count * n ** 3:
            raise ValueError("out_host must be a pinned buffer of count * n^3 doubles")
        if copy_stream is None:
            raise ValueError("streaming download needs a copy stream")
        _native.call("rbws_mgcg_solve_to_host", ctx.handle, f.data_ptr(), f_stride,
                     x.data_ptr(), float(delta), int(l_max), iters.ctypes.data,
                     hist.ctypes.data, tres.ctypes.data, status.ctypes.data,
                     _native.stream_ptr(), out_host.data_ptr(), n ** 3,
                     int(copy_stream.cuda_stream))
    else:
        _native.call("rbws_mgcg_solve", ctx.handle, f.data_ptr(), f_stride, x.data_ptr(),
                     float(delta), int(l_max), iters.ctypes.data, hist.ctypes.data,
                     tres.ctypes.data, status.ctypes.data, _native.stream_ptr())
    wall = time.perf_counter() - t0
    if raise_on_breakdown and np.any(status & 1):
        bad = int(np.flatnonzero(status & 1)[0])
        raise OperatorError(f"non-positive curvature for parameter #{bad}; operator not SPD")
    reports = SolveReports(method, iters, hist, tres, status, wall, delta, l_max, ctx.mus,
                           {"batch": count, "batch_wall_time": wall, "smoother": ctx.smoother_kind,
                            "nu": ctx.nu})
    return x, reports
