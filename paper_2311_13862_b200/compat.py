"""Reference-signature drop-in for the RBWS hot path: the ``rbws`` package's per-parameter
API (numpy vectors in the reference's free-DoF order, one parameter per call) over the
batched native path.

    from paper_2311_13862_b200 import compat as rbws      # instead of ``import rbws``

    prob = rbws.ParametricProblem(rbws.get_problem("example-1"), levels=3, m0=4)
    hf = rbws.HighFidelitySolver(prob, method="lu")
    model = rbws.l1roc_offline(train, N, hf, prob.operator, prob.operator_rows, prob.rhs)
    for mu in test:
        A, f = prob.operator(mu), prob.rhs(mu)
        ctx = rbws.mg_context_for(prob, mu)
        x, rep = rbws.rbi_pcg_solve(A, f, cfg, mg_ctx=ctx, l1roc_model=model, mu=mu)

This is the call sequence of the reference's experiment loop (experiment.py:108-172); every
name below keeps the reference's signature, argument meaning and errors:

* ``ParametricProblem(spec, levels, m0)`` (grid.py:193-290): ``operator(mu, level)``
  returns a device-backed :class:`Operator` (``A @ x``, ``A.diagonal()``, ``A[rows, :]``,
  ``A.shape``; ``tocsr()`` for assembled problems) instead of a scipy matrix — the product
  never forms the finest operator; ``operator_rows``, ``rhs``, ``system``, ``free``;
* ``mg_context_for`` / ``mg_vcycle`` / ``mgcg_solve`` (multigrid.py:191-232), ``pcg_solve`` /
  ``cg_solve`` (krylov.py:42-114, any preconditioner callable), ``rbi_pcg_solve`` /
  ``make_initial_guess`` / ``initial_residual`` / ``MethodConfig`` (warmstart.py:37-117),
  ``l1roc_offline`` / ``l1roc_online`` / ``L1rocModel`` (rb.py:134-293),
  ``HighFidelitySolver`` (hf.py:12-60), ``msrb_train`` (msrb.py:113-149),
  ``lhs_sample`` (sampling.py:8-27), ``get_problem`` (problems.py:158-162), ``SolveReport``,
  ``OperatorError``, ``DegenerateBasisError``.

Inside, each call is the batched native path with a batch of one parameter (mu-bound
contexts are cached per problem, so ``prob.operator(mu)``, ``mg_context_for(prob, mu)`` and
the solve share one device context).  Whole batches should use the batched API of the
package itself (``mg_context_for(prob, mus)``, ``rbi_pcg_solve`` on a ``BatchOperator``,
``HostPipeline``), which this module wraps.

Deviations, all documented: ``HighFidelitySolver(method="lu")`` solves by MGCG driven to
1e-14 (no sparse direct solver runs on the device; the snapshots agree with SuperLU's to
~1e-12); ``mg_vcycle`` of the padded-layout problems starts on the finest level only.
``pcg_solve`` with a preconditioner other than this module's multigrid V-cycle runs the
reference's loop with the caller's callable on the host (device operator applies); with the
V-cycle (``mg_preconditioner(ctx)``, or via ``mgcg_solve`` / ``rbi_pcg_solve``) the whole
loop is the native batched PCG.
"""

from __future__ import annotations

import time
from collections import OrderedDict

import numpy as np
import scipy.sparse as sp

from . import _native
from . import grid as _grid
from . import hf as _hf
from . import msrb as _msrb
from . import multigrid as _mg
from . import rb as _rb
from . import warmstart as _ws
from .fem import example1, example2
from .krylov import OperatorError, SolveReport
from .problems import get_problem, lhs_sample
from .rb import DegenerateBasisError, l1_indicator
from .warmstart import METHODS, MethodConfig

__all__ = [
    "ParametricProblem", "Operator", "MgContext", "mg_context_for", "mg_vcycle", "mgcg_solve",
    "mg_preconditioner", "pcg_solve", "cg_solve", "rbi_pcg_solve", "make_initial_guess",
    "initial_residual", "MethodConfig", "METHODS", "L1rocModel", "l1roc_offline",
    "l1roc_online", "l1_indicator", "HighFidelitySolver", "MsrbHierarchy", "msrb_train",
    "lhs_sample", "get_problem", "example1", "example2", "SolveReport", "OperatorError",
    "DegenerateBasisError", "AssembledSystem",
]

_CTX_CACHE = 8  # mu-bound device contexts kept per problem


def _key(mu) -> bytes:
    return np.ascontiguousarray(mu, dtype=np.float64).tobytes()


# ------------------------------------------------------------------------- problems

class AssembledSystem:
    """One parameter instance (grid.py:185-191): operator, rhs, mu, free node ids."""

    def __init__(self, operator, rhs, mu, free):
        self.operator, self.rhs, self.mu, self.free = operator, rhs, mu, free


class ParametricProblem:
    """The reference's ParametricProblem (grid.py:193-290) over the device hierarchy."""

    def __init__(self, spec, levels: int = 3, m0: int = 2):
        if isinstance(spec, str):
            spec = get_problem(spec)
        self.spec = spec
        self.native = _grid.ParametricProblem(spec, levels=levels, m0=m0)
        from .fem_fn import FnFemProblem
        self._fn = isinstance(self.native, FnFemProblem)
        self.cells = tuple(self.native.cells)
        self._ctxs: OrderedDict = OrderedDict()
        if self._fn:
            self.free_by_level = list(self.native.free_by_level)
        else:
            self.free_by_level = [self._interior(c) for c in self.cells]
        self.free = self.free_by_level[-1]
        self.n_free = len(self.free)

    @staticmethod
    def _interior(c: int) -> np.ndarray:
        i = np.arange(c + 1)
        K, J, I = np.meshgrid(i, i, i, indexing="ij")
        inner = (I > 0) & (I < c) & (J > 0) & (J < c) & (K > 0) & (K < c)
        return np.flatnonzero(inner.ravel())

    @property
    def levels(self) -> int:
        return len(self.cells)

    @property
    def finest_level(self) -> int:
        return self.levels - 1

    # -- layout: numpy free-DoF vectors <-> device vectors of the native layout
    def to_device(self, v, level: int | None = None):
        level = self.finest_level if level is None else level
        if self._fn:
            return self.native.to_full(np.asarray(v, dtype=np.float64)[None], level)
        return _grid.to_padded(np.asarray(v, dtype=np.float64), self.cells[level])

    def from_device(self, t, level: int | None = None) -> np.ndarray:
        level = self.finest_level if level is None else level
        if self._fn:
            return self.native.from_full(t.view(1, -1), level)[0].copy()
        return _grid.from_padded(t, self.cells[level], 1)[0].copy()

    def context(self, mu, nu: int = 1, smoother: str = "auto"):
        """The cached native one-instance context of mu (operators of every level, smoother
        data, coarsest factor)."""
        mu = self.spec.check_mu(mu)
        k = (_key(mu), nu, smoother)
        ctx = self._ctxs.get(k)
        if ctx is None:
            ctx = _mg.mg_context_for(self.native, mu[None], nu=nu, smoother=smoother)
            self._ctxs[k] = ctx
            while len(self._ctxs) > _CTX_CACHE:
                self._ctxs.popitem(last=False)
        else:
            self._ctxs.move_to_end(k)
        return ctx

    # -- reference API
    def operator(self, mu, level: int | None = None) -> "Operator":
        """A_h(mu) on the free DoFs of `level` (grid.py:246-255)."""
        return Operator(self, self.spec.check_mu(mu), self.finest_level if level is None else level)

    def operator_rows(self, mu, rows) -> sp.csr_matrix:
        """A_h(mu)[rows, :] (grid.py:257-264)."""
        return self.operator(mu).rows(rows)

    def rhs(self, mu) -> np.ndarray:
        """f_h(mu) on the free DoFs (grid.py:266-284)."""
        mu = self.spec.check_mu(mu)
        if hasattr(self.native, "rhs_host"):
            return np.asarray(self.native.rhs_host(mu[None])[0], dtype=np.float64).copy()
        return self.from_device(self.native.rhs(mu[None]))

    def system(self, mu) -> AssembledSystem:
        mu = self.spec.check_mu(mu)
        return AssembledSystem(self.operator(mu), self.rhs(mu), mu, self.free)


class Operator:
    """A_h(mu) at one level as a device-backed linear operator (the reference returns a
    scipy CSR; the product never stores the finest operator)."""

    def __init__(self, problem: ParametricProblem, mu, level: int):
        self.problem, self.mu, self.level = problem, mu, level
        m = len(problem.free_by_level[level])
        self.shape = (m, m)
        self.dtype = np.dtype(np.float64)

    def _ctx(self):
        return self.problem.context(self.mu)

    def _apply_dev(self, t):
        ctx = self._ctx()
        if self.problem._fn:
            return ctx.apply(t, self.level)
        return _grid.BatchOperator(ctx).apply(t, self.level)

    def __matmul__(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 2:
            return np.column_stack([self @ x[:, j] for j in range(x.shape[1])])
        if x.shape != (self.shape[1],):
            raise ValueError("dimension mismatch")
        p = self.problem
        return p.from_device(self._apply_dev(p.to_device(x, self.level)), self.level)

    dot = __matmul__

    def diagonal(self) -> np.ndarray:
        p = self.problem
        ctx = self._ctx()
        if p._fn:
            c = p.cells[self.level]
            nodes = (c + 1) ** 3
            dg = ctx.coefA[self.level][: 27 * nodes].view(27, nodes)[13]
            return dg.cpu().numpy()[p.free_by_level[self.level]].copy()
        if self.level == 0:
            return np.diag(self.toarray()).copy()
        import torch
        c = p.cells[self.level]
        out = torch.zeros(_grid.padded_len(c, 1), dtype=torch.float64, device="cuda")
        _native.call("rbws_batch_dinv", ctx.handle, self.level, out.data_ptr(),
                     _native.stream_ptr())
        return 1.0 / p.from_device(out, self.level)

    def rows(self, rows) -> sp.csr_matrix:
        """A[rows, :] from operator applies to unit vectors (A is symmetric)."""
        rows = np.asarray(list(rows), dtype=np.int64)
        out = []
        for r in rows:
            e = np.zeros(self.shape[1])
            e[r] = 1.0
            out.append(sp.csr_matrix(self @ e))
        if not out:
            return sp.csr_matrix((0, self.shape[1]))
        M = sp.vstack(out).tocsr()
        M.eliminate_zeros()
        return M

    def __getitem__(self, key):
        if isinstance(key, tuple) and len(key) == 2 and key[1] == slice(None):
            return self.rows(np.atleast_1d(key[0]))
        raise TypeError("Operator supports A[rows, :] only")

    def tocsr(self) -> sp.csr_matrix:
        """The assembled matrix: host operators of assembled problems; for the matrix-free
        FV problems columns are applied (small grids only)."""
        nat = self.problem.native
        if hasattr(nat, "operator_host"):
            return nat.operator_host(self.mu, self.level).tocsr()
        if self.shape[0] > 30000:
            raise MemoryError("matrix-free operator too large to assemble; use A @ x")
        cols = [sp.csr_matrix(self @ e).T for e in np.eye(self.shape[0])]
        return sp.hstack(cols).tocsr()

    def toarray(self) -> np.ndarray:
        return self.tocsr().toarray()


# ------------------------------------------------------------------------- multigrid

class MgContext:
    """Per-parameter multigrid context (multigrid.py:116-129) on the device."""

    def __init__(self, problem: ParametricProblem, mu, nu: int, smoother: str):
        self.problem, self.mu, self.nu = problem, mu, nu
        self.native = problem.context(mu, nu, smoother)
        self.smoother_kind = (getattr(self.native, "smoother", None)
                              or getattr(self.native, "smoother_kind", smoother))

    @property
    def levels(self) -> int:
        return self.problem.levels

    @property
    def operators(self) -> tuple:
        return tuple(Operator(self.problem, self.mu, l) for l in range(self.levels))


def mg_context_for(problem: ParametricProblem, mu, nu: int = 1, smoother: str = "auto"):
    """Context build from the problem's precoarsened affine terms (multigrid.py:191-202)."""
    return MgContext(problem, problem.spec.check_mu(mu), nu, smoother)


def mg_vcycle(b, ctx: MgContext, level: int | None = None) -> np.ndarray:
    """One V-cycle for A^level u = b from zero (multigrid.py:205-222)."""
    p = ctx.problem
    level = p.finest_level if level is None else level
    if not 0 <= level < ctx.levels:
        raise ValueError(f"level {level} outside hierarchy")
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != len(p.free_by_level[level]):
        raise ValueError("right-hand side does not match level size")
    if p._fn:
        return p.from_device(ctx.native.vcycle(p.to_device(b, level), level), level)
    if level != p.finest_level:
        raise ValueError("the device V-cycle of this problem starts on the finest level")
    return p.from_device(_mg.mg_vcycle(p.to_device(b), ctx.native))


class _MgPrecond:
    """``lambda r, k: mg_vcycle(r, ctx)`` that pcg_solve recognises (native PCG loop)."""

    def __init__(self, ctx: MgContext):
        self.ctx = ctx

    def __call__(self, r, k):
        return mg_vcycle(r, self.ctx)


def mg_preconditioner(ctx: MgContext) -> _MgPrecond:
    return _MgPrecond(ctx)


def _report(rep, mu, wall, method=None) -> SolveReport:
    rep.mu = None if mu is None else np.asarray(mu, dtype=np.float64)
    rep.wall_time = wall
    if method is not None:
        rep.method = method
    return rep


def _native_pcg(ctx: MgContext, f, x0, delta, l_max, mu, method):
    import torch
    p = ctx.problem
    t0 = time.perf_counter()
    fd = p.to_device(f)
    xd = p.to_device(np.zeros(len(f)) if x0 is None else x0)
    if p._fn:
        from . import fem_fn
        x, reps = fem_fn.mgcg_solve(ctx.native, fd, xd, delta=delta, l_max=l_max, method=method)
    else:
        x, reps = _mg.mgcg_solve(None, fd, xd, ctx.native, delta=delta, l_max=l_max,
                                 method=method, overwrite_x0=True)
    out = p.from_device(x)
    torch.cuda.synchronize()
    return out, _report(reps[0], mu, time.perf_counter() - t0)


def _same_operator(A, ctx: MgContext) -> bool:
    return (isinstance(A, Operator) and A.problem is ctx.problem
            and A.level == ctx.problem.finest_level and _key(A.mu) == _key(ctx.mu))


def mgcg_solve(A, f, x0, ctx: MgContext, delta: float = 1e-16, l_max: int = 40, mu=None,
               method: str = "mgcg"):
    """PCG with one V-cycle per preconditioner application (multigrid.py:225-232)."""
    return pcg_solve(A, f, x0, precond=mg_preconditioner(ctx), delta=delta, l_max=l_max,
                     method=method, mu=mu)


def pcg_solve(A, f, x0, precond=None, delta: float = 1e-16, l_max: int = 40,
              method: str = "pcg", mu=None):
    """Preconditioned CG for SPD A (krylov.py:42-109).  With this module's V-cycle on the
    context of A the whole loop runs natively; otherwise the reference's loop runs with
    the caller's preconditioner callable (A applied on the device when it is an
    :class:`Operator`)."""
    if delta <= 0:
        raise ValueError("tolerance must be positive")
    if l_max < 0:
        raise ValueError("l_max must be non-negative")
    if isinstance(precond, _MgPrecond) and _same_operator(A, precond.ctx):
        return _native_pcg(precond.ctx, np.asarray(f, dtype=np.float64), x0, delta, l_max,
                           mu, method)
    t0 = time.perf_counter()
    f = np.asarray(f, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    fnorm = np.linalg.norm(f)
    absolute = fnorm == 0.0
    scale = 1.0 if absolute else fnorm

    def apply_p(r, k):
        if precond is None:
            return r.copy()
        s = precond(r, k)
        return s.copy() if s is r else s

    r = f - A @ x
    history = [float(np.linalg.norm(r) / scale)]
    k = 0
    if history[0] > delta and l_max > 0:
        s = apply_p(r, 0)
        p = s
        rs = float(r @ s)
        while k < l_max:
            Ap = A @ p
            pAp = float(p @ Ap)
            if pAp <= 0.0:
                raise OperatorError(f"non-positive curvature p.A.p = {pAp:g}; operator not SPD")
            alpha = rs / pAp
            x += alpha * p
            r -= alpha * Ap
            k += 1
            relres = float(np.linalg.norm(r) / scale)
            history.append(relres)
            if relres <= delta:
                break
            s = apply_p(r, k)
            rs_new = float(r @ s)
            beta = rs_new / rs
            p = s + beta * p
            rs = rs_new
    true_res = float(np.linalg.norm(f - A @ x) / scale)
    return x, SolveReport(method, k, history, true_res <= delta, true_res,
                          time.perf_counter() - t0, delta, l_max,
                          None if mu is None else np.asarray(mu, dtype=np.float64), absolute)


def cg_solve(A, f, x0, delta: float = 1e-16, l_max: int = 40, mu=None):
    """Plain CG: PCG with the identity preconditioner (krylov.py:112-114)."""
    return pcg_solve(A, f, x0, None, delta, l_max, method="cg", mu=mu)


# ------------------------------------------------------------------------- RB models

class L1rocModel:
    """Trained over-collocation model (rb.py:134-175) with its device-resident basis."""

    def __init__(self, native: _rb.L1rocModel, problem: ParametricProblem | None = None):
        self.native, self.problem = native, problem
        self._basis = None

    @property
    def basis(self) -> np.ndarray:
        if self._basis is None:
            self._basis = self.native.basis_numpy()
        return self._basis

    transform = property(lambda self: self.native.transform)
    collocation = property(lambda self: self.native.collocation)
    solution_points = property(lambda self: self.native.solution_points)
    residual_points = property(lambda self: self.native.residual_points)
    chosen_mus = property(lambda self: self.native.chosen_mus)
    indicator_history = property(lambda self: self.native.indicator_history)
    saturated = property(lambda self: self.native.saturated)
    dim = property(lambda self: self.native.dim)
    n_points = property(lambda self: self.native.n_points)

    def prefix(self, N: int) -> "L1rocModel":
        return L1rocModel(self.native.prefix(N), self.problem)


class HighFidelitySolver:
    """Per-parameter high-fidelity solver (hf.py:12-60).  ``method="lu"`` is served by
    MGCG driven to 1e-14 (no sparse direct solver on the device)."""

    def __init__(self, problem: ParametricProblem, method: str = "lu", delta: float = 1e-14,
                 l_max: int = 100, nu: int = 1, smoother: str = "auto", max_cached: int = 128):
        if method not in ("lu", "mgcg"):
            raise ValueError(f"unknown high-fidelity method {method!r}")
        self.problem, self.method = problem, method
        self.delta = min(delta, 1e-14) if method == "lu" else delta
        self.l_max = max(l_max, 200) if method == "lu" else l_max
        self.nu, self.smoother, self.max_cached = nu, smoother, max_cached
        self.native = _hf.HighFidelitySolver(problem.native, delta=self.delta, l_max=self.l_max,
                                             nu=nu, smoother=smoother)

    def solve_device(self, mu, rhs=None):
        return self.native.solve(np.asarray(mu, dtype=np.float64),
                                 None if rhs is None else self.problem.to_device(rhs))

    def solve(self, mu, rhs=None) -> np.ndarray:
        x = self.solve_device(mu, rhs)
        return self.problem.from_device(x)

    def __call__(self, mu, rhs=None) -> np.ndarray:
        return self.solve(mu, rhs)


def _bound_problem(fn, what: str) -> ParametricProblem:
    prob = getattr(fn, "__self__", None)
    if not isinstance(prob, ParametricProblem):
        raise TypeError(f"{what} must be a bound method of a compat ParametricProblem "
                        "(the device path needs the problem's affine terms)")
    return prob


def l1roc_offline(mus, N: int, hf_solve, operator, operator_rows, rhs, seed: int = 0):
    """Greedy over-collocation training (rb.py:208-293), reference signature."""
    prob = _bound_problem(operator, "operator")
    for fn, name in ((operator_rows, "operator_rows"), (rhs, "rhs")):
        if _bound_problem(fn, name) is not prob:
            raise TypeError(f"{name} belongs to a different problem")
    if isinstance(hf_solve, HighFidelitySolver):
        hf = hf_solve.native
    else:
        hf = lambda mu: prob.to_device(hf_solve(mu))  # noqa: E731
    mus = np.asarray([np.asarray(m, dtype=np.float64) for m in mus])
    model = _rb.l1roc_offline(mus, N, hf, prob.native, seed=seed)
    return L1rocModel(model, prob)


def l1roc_online(model: L1rocModel, A, b):
    """Sub-sampled least-squares reduced solve (rb.py:190-205); A: a problem's Operator."""
    if model.dim == 0:
        raise ValueError("empty model")
    if not isinstance(A, Operator):
        raise TypeError("A must be a compat Operator (prob.operator(mu))")
    p = A.problem
    u0, c = _rb.l1roc_online(model.native, _grid.BatchOperator(A._ctx()), p.to_device(b))
    return p.from_device(u0), np.asarray(c[0])


class MsrbHierarchy:
    """Trained multispace hierarchy (msrb.py:88-110)."""

    def __init__(self, native):
        self.native = native

    def __getattr__(self, name):
        return getattr(self.native, name)


def msrb_train(mus, N: int, K_max: int, hf_solver, operator, rhs) -> MsrbHierarchy:
    """Per-iteration error-snapshot bases (msrb.py:113-149), reference signature."""
    prob = _bound_problem(operator, "operator")
    if not isinstance(hf_solver, HighFidelitySolver):
        raise TypeError("hf_solver must be a compat HighFidelitySolver")
    mus = np.asarray([np.asarray(m, dtype=np.float64) for m in mus])
    return MsrbHierarchy(_msrb.msrb_train(mus, N, K_max, hf_solver.native, prob.native))


# ------------------------------------------------------------------------- warm starts

def initial_residual(A, f, u0) -> float:
    """||f - A u0|| / ||f|| (warmstart.py:63-68)."""
    f = np.asarray(f, dtype=np.float64)
    r = f - A @ np.asarray(u0, dtype=np.float64)
    fn = np.linalg.norm(f)
    return float(np.linalg.norm(r) / (fn if fn > 0 else 1.0))


def make_initial_guess(A, f, cfg: MethodConfig, l1roc_model: L1rocModel | None = None,
                       msrb_hier: MsrbHierarchy | None = None) -> np.ndarray:
    """Initial guess per the method pairing (warmstart.py:71-85)."""
    if cfg.initializer == "zero":
        return np.zeros(len(f))
    if cfg.initializer == "l1roc":
        if l1roc_model is None:
            raise ValueError(f"{cfg.method} requires a trained over-collocation model")
        model = l1roc_model if cfg.N in (0, l1roc_model.dim) else l1roc_model.prefix(cfg.N)
        u0, _ = l1roc_online(model, A, f)
        return u0
    if cfg.initializer == "pod":
        if msrb_hier is None:
            raise ValueError(f"{cfg.method} requires a trained multispace hierarchy")
        # POD Galerkin solve (rb.py:71-83): W^T A W a = W^T f on the basis of the hierarchy
        W = msrb_hier.native.init_basis.basis
        n = A.problem.native.n
        Wn = W[:, : n ** 3].reshape(-1, n, n, n)[:, 1:, 1:, 1:].reshape(W.shape[0], -1)
        Wn = Wn.T.cpu().numpy()
        a = np.linalg.solve(Wn.T @ (A @ Wn), Wn.T @ np.asarray(f, dtype=np.float64))
        return Wn @ a
    raise ValueError(f"unknown initializer {cfg.initializer!r}")


def rbi_pcg_solve(A, f, cfg: MethodConfig, mg_ctx: MgContext | None = None,
                  l1roc_model: L1rocModel | None = None, msrb_hier: MsrbHierarchy | None = None,
                  mu=None, residual_log: list | None = None):
    """Initialise per the method pairing, then refine with one PCG run
    (warmstart.py:88-117)."""
    import torch
    f = np.asarray(f, dtype=np.float64)
    extra = dict(N=cfg.N, nu=cfg.nu, smoother=cfg.smoother, K_max=cfg.K_max,
                 initializer=cfg.initializer, preconditioner=cfg.preconditioner,
                 config_hash=cfg.config_hash())
    if cfg.preconditioner == "mg":
        if mg_ctx is None:
            raise ValueError("multigrid preconditioning requires a context")
        if cfg.initializer == "l1roc" and l1roc_model is None:
            raise ValueError(f"{cfg.method} requires a trained over-collocation model")
        p = mg_ctx.problem
        if residual_log is None and _same_operator(A, mg_ctx):
            t0 = time.perf_counter()
            model = None if l1roc_model is None else l1roc_model.native
            x, reps = _ws.rbi_pcg_solve(_grid.BatchOperator(mg_ctx.native), p.to_device(f),
                                        cfg, mg_ctx=mg_ctx.native, l1roc_model=model)
            out = p.from_device(x)
            torch.cuda.synchronize()
            rep = _report(reps[0], mu, time.perf_counter() - t0, cfg.method)
            rep.config.update(extra)
            return out, rep
        u0 = make_initial_guess(A, f, cfg, l1roc_model, msrb_hier)
        precond = mg_preconditioner(mg_ctx)
    elif cfg.preconditioner == "msrb":
        if msrb_hier is None:
            raise ValueError("msrb preconditioning requires a trained hierarchy")
        if residual_log is not None or not isinstance(A, Operator):
            raise NotImplementedError("rbi-msrbcg runs natively on the problem's operator only")
        p = A.problem
        t0 = time.perf_counter()
        x, reps = _msrb.rbi_msrbcg_solve(p.native, A.mu[None], msrb_hier.native,
                                         f=p.to_device(f), delta=cfg.delta, l_max=cfg.l_max,
                                         method=cfg.method)
        out = p.from_device(x.reshape(-1)[: p.native.n ** 3].contiguous())
        torch.cuda.synchronize()
        rep = _report(reps[0], mu, time.perf_counter() - t0, cfg.method)
        rep.config.update(extra)
        return out, rep
    else:
        raise ValueError(f"unknown preconditioner {cfg.preconditioner!r}")
    if residual_log is not None:
        inner = precond
        precond = lambda r, k: (residual_log.append(r.copy()), inner(r, k))[1]  # noqa: E731
    x, rep = pcg_solve(A, f, u0, precond=precond, delta=cfg.delta, l_max=cfg.l_max,
                       method=cfg.method, mu=mu)
    rep.config.update(extra)
    return x, rep
