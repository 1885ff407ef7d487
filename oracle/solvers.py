"""Oracle solvers — TEST INFRASTRUCTURE ONLY.

numpy/scipy restatement of the reference's solver path (file:line in each
docstring refers to /root/reference/pkg/src/rbws).  Used by tests as the
checker and by bench.py as the timed CPU baseline; never by the product.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

JACOBI_OMEGA = 0.7   # multigrid.py:27
PLANE_OMEGA = 0.6    # multigrid.py:29 (damped plane-Jacobi of the anisotropic problem)


class OperatorError(Exception):
    pass


class DegenerateBasisError(Exception):
    pass


# ----------------------------------------------------------------- grid / MG

def galerkin(A_fine, P) -> sp.csr_matrix:
    """P^T A P (grid.py:173-182)."""
    A_fine = sp.csr_matrix(A_fine)
    P = sp.csr_matrix(P)
    if A_fine.shape[1] != P.shape[0]:
        raise ValueError("incompatible shapes for coarsening")
    return (P.T @ (A_fine @ P)).tocsr()


def jacobi_sweep(A, diag, x, b, omega=JACOBI_OMEGA):
    """One damped Jacobi sweep x + omega (b - A x)/diag (kernels.py:98-115)."""
    return x + omega * (b - A @ x) / diag


def gs_sweep(A, x, b, forward: bool = True):
    """One in-place Gauss-Seidel sweep (reference _smoothers.pyx:14-28 csr_gauss_seidel,
    kernels.py:117-129): x_i = (b_i - sum_{j != i} a_ij x_j) / a_ii row by row, rows in
    ascending (forward) or descending (backward) order.  Vectorised as the triangular
    solve of the reference's NumPy backend (_smoothers_np.py:35-42), which is the same
    sequential update."""
    from scipy.sparse.linalg import spsolve_triangular
    A = sp.csr_matrix(A)
    if forward:
        x[:] = spsolve_triangular(sp.csr_matrix(sp.tril(A, k=0)),
                                  b - sp.triu(A, k=1) @ x, lower=True)
    else:
        x[:] = spsolve_triangular(sp.csr_matrix(sp.triu(A, k=0)),
                                  b - sp.tril(A, k=-1) @ x, lower=False)
    return x


class PlaneSmoother:
    """z-plane block smoother (multigrid.py:48-110): plane blocks A[plane, plane] solved
    exactly by sparse LU (scipy splu, as the reference), neighbour couplings only to the adjacent layers.  omega = 1:
    block Gauss-Seidel, ascending planes before / descending after the coarse correction
    ("plane-z"); omega < 1: damped block Jacobi x += omega A_pp^-1 (b - A x)_p
    ("plane-jacobi")."""

    def __init__(self, A, layers, omega: float = 1.0):
        A = sp.csr_matrix(A)
        layers = np.asarray(layers)
        if len(layers) != A.shape[0]:
            raise ValueError("layer map does not match operator size")
        self.A, self.omega = A, float(omega)
        self.planes = [np.flatnonzero(layers == z) for z in np.unique(layers)]
        self.factors, self.nbrs = [], []
        for p, idx in enumerate(self.planes):
            try:
                self.factors.append(spla.splu(A[idx][:, idx].tocsc()))
            except RuntimeError as exc:
                raise OperatorError(f"plane block singular: {exc}") from exc
            prv = A[idx][:, self.planes[p - 1]].tocsr() if p > 0 else None
            nxt = A[idx][:, self.planes[p + 1]].tocsr() if p + 1 < len(self.planes) else None
            self.nbrs.append((prv, nxt))

    def _gs(self, x, b, order):
        for p in order:
            idx = self.planes[p]
            rhs = b[idx].copy()
            prv, nxt = self.nbrs[p]
            if prv is not None:
                rhs -= prv @ x[self.planes[p - 1]]
            if nxt is not None:
                rhs -= nxt @ x[self.planes[p + 1]]
            x[idx] = self.factors[p].solve(rhs)
        return x

    def _jacobi(self, x, b):
        r = b - self.A @ x
        for p, idx in enumerate(self.planes):
            x[idx] += self.omega * self.factors[p].solve(r[idx])
        return x

    def sweep(self, u, b, nu, forward: bool):
        x = np.array(u, dtype=np.float64, copy=True)
        order = range(len(self.planes)) if forward else range(len(self.planes) - 1, -1, -1)
        for _ in range(nu):
            x = self._gs(x, b, order) if self.omega == 1.0 else self._jacobi(x, b)
        return x


def default_smoother(problem) -> str:
    """Plane smoothing when any term is anisotropic, damped Jacobi otherwise
    (multigrid.py:183-188)."""
    aniso = getattr(problem.spec, "aniso", ())
    return "plane-jacobi" if any(len(set(a)) > 1 for a in aniso) else "jacobi"


@dataclass
class OracleMgContext:
    """Per-parameter V-cycle data (multigrid.py:116-129, 154-168)."""

    operators: list
    prolongations: list
    diags: list
    nu: int
    coarse_factor: tuple
    omega: float = JACOBI_OMEGA
    smoother: str = "jacobi"  # "jacobi" (isotropic default) or "gs" (multigrid.py:132-152)
    planes: list | None = None  # PlaneSmoother per level ("plane-z" / "plane-jacobi")

    @property
    def levels(self):
        return len(self.operators)


def mg_context_for(problem, mu, nu: int = 1, omega: float = JACOBI_OMEGA,
                   smoother: str = "jacobi") -> OracleMgContext:
    """Operators per level from the affine terms + Cholesky of level 0 (multigrid.py:191-202)."""
    if nu < 0:
        raise ValueError("smoothing count must be non-negative")
    ops = [problem.operator(mu, level=i) for i in range(problem.levels)]
    try:
        cf = sla.cho_factor(ops[0].toarray())
    except sla.LinAlgError as exc:
        raise OperatorError(f"coarsest operator not SPD: {exc}") from exc
    if smoother == "auto":
        smoother = default_smoother(problem)
    diags = [A.diagonal().copy() for A in ops]
    if smoother in ("plane-z", "plane-jacobi"):
        layers = getattr(problem, "layers_by_level", None)
        if layers is None:
            raise ValueError("plane smoothing needs per-level layer maps")
        w = 1.0 if smoother == "plane-z" else PLANE_OMEGA
        planes = [None] + [PlaneSmoother(ops[i], layers[i], w) for i in range(1, len(ops))]
        return OracleMgContext(ops, list(problem.prolongations), diags, nu, cf, w, smoother,
                               planes)
    for d in diags[1:]:
        if np.any(d == 0.0):
            raise ValueError("zero diagonal entry; point smoothing undefined")
    if smoother not in ("jacobi", "gs"):
        raise ValueError(f"unknown smoother kind {smoother!r}")
    return OracleMgContext(ops, list(problem.prolongations), diags, nu, cf, omega, smoother)


def mg_vcycle(b, ctx: OracleMgContext, level=None) -> np.ndarray:
    """One V-cycle from zero (multigrid.py:205-222) with Jacobi pre/post sweeps."""
    if level is None:
        level = ctx.levels - 1
    b = np.asarray(b, dtype=np.float64)
    if level == 0:
        return sla.cho_solve(ctx.coarse_factor, b)
    A, d = ctx.operators[level], ctx.diags[level]
    P = ctx.prolongations[level - 1]
    if ctx.planes is not None:  # plane smoothers (multigrid.py:97-110, 219-222)
        sm = ctx.planes[level]
        u = sm.sweep(np.zeros_like(b), b, ctx.nu, True)
        e = mg_vcycle(P.T @ (b - A @ u), ctx, level - 1)
        return sm.sweep(u + P @ e, b, ctx.nu, False)
    u = np.zeros_like(b)
    for _ in range(ctx.nu):  # "gs": forward sweeps before, backward after (multigrid.py:137-138)
        u = jacobi_sweep(A, d, u, b, ctx.omega) if ctx.smoother == "jacobi" else gs_sweep(A, u, b, True)
    r = b - A @ u
    e = mg_vcycle(P.T @ r, ctx, level - 1)
    u = u + P @ e
    for _ in range(ctx.nu):
        u = jacobi_sweep(A, d, u, b, ctx.omega) if ctx.smoother == "jacobi" else gs_sweep(A, u, b, False)
    return u


# ---------------------------------------------------------------------- PCG

@dataclass
class SolveReport:
    """Convergence record (krylov.py:25-39)."""

    method: str
    iterations: int
    history: list
    converged: bool
    true_residual: float
    wall_time: float
    delta: float
    l_max: int
    mu: np.ndarray | None = None
    absolute_norms: bool = False
    config: dict = field(default_factory=dict)


def pcg_solve(A, f, x0, precond=None, delta=1e-16, l_max=40, method="pcg", mu=None):
    """Preconditioned CG, recurrence residual drives the loop (krylov.py:42-109)."""
    if delta <= 0:
        raise ValueError("tolerance must be positive")
    if l_max < 0:
        raise ValueError("l_max must be non-negative")
    t0 = time.perf_counter()
    f = np.asarray(f, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    fn = np.linalg.norm(f)
    absolute = fn == 0.0
    scale = 1.0 if absolute else fn
    prec = (lambda r, k: r.copy()) if precond is None else precond
    r = f - A @ x
    hist = [float(np.linalg.norm(r) / scale)]
    k = 0
    if hist[0] > delta and l_max > 0:
        s = prec(r, 0)
        p = s.copy()
        rs = float(r @ s)
        while k < l_max:
            q = A @ p
            pq = float(p @ q)
            if pq <= 0.0:
                raise OperatorError(f"non-positive curvature p.A.p = {pq:g}; operator not SPD")
            alpha = rs / pq
            x += alpha * p
            r -= alpha * q
            k += 1
            rel = float(np.linalg.norm(r) / scale)
            hist.append(rel)
            if rel <= delta:
                break
            s = prec(r, k)
            rs_new = float(r @ s)
            beta = rs_new / rs
            p = s + beta * p
            rs = rs_new
    tr = float(np.linalg.norm(f - A @ x) / scale)
    return x, SolveReport(method, k, hist, tr <= delta, tr, time.perf_counter() - t0,
                          delta, l_max, None if mu is None else np.asarray(mu, float), absolute)


def mgcg_solve(A, f, x0, ctx, delta=1e-16, l_max=40, mu=None, method="mgcg"):
    """PCG with one V-cycle per application (multigrid.py:225-232)."""
    return pcg_solve(A, f, x0, lambda r, k: mg_vcycle(r, ctx), delta, l_max, method, mu)


# ------------------------------------------------------------------- L1ROC

def deim_extend(W, X, v, exclude=None):
    """Interpolatory basis extension (rb.py:96-126).

    Returns (column, index, coeffs, pivot).
    """
    v = np.asarray(v, dtype=np.float64)
    W = np.zeros((len(v), 0)) if W is None else np.asarray(W)
    X = list(X)
    if W.shape[1] != len(X):
        raise ValueError("basis width and point count differ")
    if W.shape[1] == 0:
        c = np.zeros(0)
        rho = v.copy()
    else:
        c = np.linalg.solve(W[X, :], v[X])
        rho = v - W @ c
    if np.max(np.abs(rho)) <= 1e-14 * max(np.max(np.abs(v)), 1e-300):
        raise DegenerateBasisError("snapshot numerically inside the current basis")
    mag = np.abs(rho)
    if exclude:
        mag = mag.copy()
        mag[list(exclude)] = -1.0
    idx = int(np.argmax(mag))
    piv = rho[idx]
    if piv == 0.0:
        raise DegenerateBasisError("residual vanishes at all admissible points")
    return rho / piv, idx, c, piv


def l1_indicator(c) -> float:
    """||c||_1 (rb.py:129-131)."""
    return float(np.sum(np.abs(np.asarray(c))))


def _lstsq(B, b):
    """Least squares with rank check (rb.py:182-187)."""
    a, _, rank, _ = np.linalg.lstsq(B, b, rcond=None)
    if rank < B.shape[1]:
        raise DegenerateBasisError("sub-sampled reduced system is rank deficient")
    return a


@dataclass(frozen=True)
class OracleL1rocModel:
    """Trained over-collocation model (rb.py:134-175)."""

    basis: np.ndarray
    transform: np.ndarray
    collocation: np.ndarray
    solution_points: np.ndarray
    residual_points: np.ndarray
    chosen: np.ndarray          # indices into the training list
    indicator_history: np.ndarray
    saturated: bool = False

    @property
    def dim(self):
        return self.basis.shape[1]

    def prefix(self, N):
        if not 1 <= N <= self.dim:
            raise ValueError("prefix dimension outside model")
        return OracleL1rocModel(self.basis[:, :N], self.transform[:N, :N],
                                self.collocation[:2 * N - 1], self.solution_points[:N],
                                self.residual_points[:N - 1], self.chosen[:N],
                                self.indicator_history[:N], self.saturated)


def l1roc_online(model: OracleL1rocModel, A, b):
    """Sub-sampled least-squares reduced solve (rb.py:190-205)."""
    if model.dim == 0:
        raise ValueError("empty model")
    rows = model.collocation
    R = A(rows) if callable(A) else A[rows, :]
    B = np.asarray(R @ model.basis)
    a = _lstsq(B, np.asarray(b, dtype=np.float64)[rows])
    return model.basis @ a, sla.solve_triangular(model.transform, a, lower=False), a


def l1roc_offline(mus, N, hf_solve, operator, operator_rows, rhs, seed=0, on_degenerate="raise"):
    """Greedy over-collocation training (rb.py:208-293).

    on_degenerate="stop" ends the greedy (flagged saturated) instead of raising
    when a picked snapshot is numerically inside the basis (bench harness only).
    """
    mus = [np.asarray(m, dtype=np.float64) for m in mus]
    if not 1 <= N <= len(mus):
        raise ValueError("need 1 <= N <= number of training parameters")
    first = int(np.random.default_rng(seed).integers(len(mus)))
    rhss = [rhs(m) for m in mus]
    n_h = len(rhss[0])
    col, idx, _, piv = deim_extend(None, [], hf_solve(mus[first]))
    W = col[:, None]
    T = np.array([[piv]])
    xs, xr, xi = [idx], [], [idx]
    chosen = [first]
    R = np.zeros((n_h, 0))
    hist = [1.0]
    saturated = False
    sampled = [operator_rows(m, xi) for m in mus]
    for _n in range(2, N + 1):
        taken = set(xs) | set(xr)
        ind = np.empty(len(mus))
        coeffs = []
        for j in range(len(mus)):
            a = _lstsq(np.asarray(sampled[j] @ W), rhss[j][xi])
            coeffs.append(a)
            ind[j] = l1_indicator(sla.solve_triangular(T, a, lower=False))
        pick = int(np.argmax(ind))
        hist.append(float(ind[pick]))
        if pick in chosen:
            saturated = True
            break
        chosen.append(pick)
        try:
            col, idx, c, piv = deim_extend(W, xs, hf_solve(mus[pick]), exclude=taken)
        except DegenerateBasisError:
            if on_degenerate != "stop":
                raise
            chosen.pop()
            saturated = True
            break
        taken.add(idx)
        T = np.block([[T, c[:, None]], [np.zeros((1, T.shape[1])), np.array([[piv]])]])
        W = np.column_stack([W, col])
        xs.append(idx)
        r = rhss[pick] - operator(mus[pick]) @ (W[:, :-1] @ coeffs[pick])
        rcol, ridx, _, _ = deim_extend(R, xr, r, exclude=taken)
        R = np.column_stack([R, rcol])
        xr.append(ridx)
        xi.extend([idx, ridx])
        for j, m in enumerate(mus):
            sampled[j] = sp.vstack([sampled[j], operator_rows(m, xi[-2:])]).tocsr()
    return OracleL1rocModel(W, T, np.asarray(xi, np.int64), np.asarray(xs, np.int64),
                            np.asarray(xr, np.int64), np.asarray(chosen, np.int64),
                            np.asarray(hist), saturated)


def rbi_mgcg_solve(problem, mu, model, delta=1e-10, l_max=40, nu=1, smoother="jacobi"):
    """RBI-MGCG: L1ROC warm start then MGCG (warmstart.py:88-117, experiment.py:149-157)."""
    A, f = problem.operator(mu), problem.rhs(mu)
    ctx = mg_context_for(problem, mu, nu=nu, smoother=smoother)
    u0 = np.zeros_like(f) if model is None else l1roc_online(model, A, f)[0]
    return mgcg_solve(A, f, u0, ctx, delta, l_max, mu,
                      "mgcg" if model is None else "rbi-mgcg")


def lhs_sample(p, n, bounds, seed=0):
    """Seeded Latin hypercube (sampling.py:8-27)."""
    if n < 1:
        raise ValueError("need at least one sample")
    bounds = np.asarray(bounds, dtype=np.float64)
    lo, hi = bounds[:, 0], bounds[:, 1]
    if np.any(hi <= lo):
        raise ValueError("degenerate bounds")
    rng = np.random.default_rng(seed)
    u = (rng.random((n, p)) + np.stack([rng.permutation(n) for _ in range(p)], axis=1)) / n
    pts = lo + u * (hi - lo)
    return [pts[i].copy() for i in range(n)]
