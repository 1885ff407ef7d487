"""L1ROC over-collocation reduced model on the B200 (reference rb.py).

* ``l1roc_online`` (rb.py:190-205) runs batched: the sampled reduced matrix
  B(mu) = A(mu)[X, :] W is assembled affinely, B(mu) = sum_q theta_q(mu) B_q,
  from the term projections B_q = (A_q W)[X, :] (computed once per model on
  the device), then every instance's M x N least-squares problem, its
  snapshot coordinates T^{-1} a and the L1 indicator are solved in one kernel
  (one CTA per instance), and the warm starts W a are expanded in one kernel.
* ``l1roc_offline`` (rb.py:208-293) keeps the reference's greedy control
  flow on the host (it is inherently sequential) while every step's data
  work — the indicator sweep over the whole training set, the high-fidelity
  solve, DEIM residuals/argmax, the residual snapshot — runs on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .grid import (ParametricProblem, interior_to_padded_index, padded_len,
                   padded_to_interior_index)


class DegenerateBasisError(Exception):
    """A snapshot or reduced operator was numerically dependent/singular."""


# ----------------------------------------------------------------- vector layouts

class PaddedLayout:
    """Interior (Dirichlet) problems: n^3 padded block per instance (grid.py layout)."""

    full_node = False

    def __init__(self, n: int):
        self.side = n
        self.S = n ** 3

    def to_storage(self, idx) -> np.ndarray:
        return interior_to_padded_index(idx, self.side)

    def from_storage(self, p) -> np.ndarray:
        return padded_to_interior_index(p, self.side)

    def free_view(self, t, count: int):
        n = self.side
        return t[: count * self.S].view(count, n, n, n)[:, 1:, 1:, 1:].reshape(count, -1)


class FullNodeLayout:
    """Problems with free boundary nodes (example-2): all (c+1)^3 nodes per instance,
    Dirichlet nodes held at zero (fem_fn.py); free DoFs are the nodes ``free`` in order."""

    full_node = True

    def __init__(self, side: int, free: np.ndarray):
        self.side = side
        self.S = side ** 3
        self.free = np.asarray(free, dtype=np.int64)

    def to_storage(self, idx) -> np.ndarray:
        return self.free[np.asarray(idx, dtype=np.int64)]

    def from_storage(self, p) -> np.ndarray:
        p = np.asarray(p, dtype=np.int64)
        i = np.searchsorted(self.free, p)
        if np.any(i >= len(self.free)) or np.any(self.free[np.minimum(i, len(self.free) - 1)] != p):
            raise ValueError("storage index is not a free node")
        return i

    def free_view(self, t, count: int):
        import torch
        fr = torch.as_tensor(self.free, device=t.device)
        return t[: count * self.S].view(count, self.S)[:, fr]


def layout_of(problem):
    from .fem_fn import FnFemProblem
    if isinstance(problem, FnFemProblem):
        return FullNodeLayout(problem.cells[-1] + 1, problem.free_by_level[-1])
    return PaddedLayout(problem.n)


def _vec(lay, count: int):
    import torch
    return torch.zeros(count * lay.S + 2 * lay.side ** 2, dtype=torch.float64, device="cuda")


def l1_indicator(c) -> float:
    """l1 norm of snapshot coordinates (rb.py:129-131)."""
    return float(np.sum(np.abs(np.asarray(c))))


@dataclass
class L1rocModel:
    """Trained over-collocation model with a device-resident basis (rb.py:134-175).

    ``basis`` is a padded tensor holding N finest-level columns back to back
    (column c at [c*n^3, (c+1)*n^3)); ``collocation`` etc. use the reference's
    free-DoF indices.
    """

    n: int
    basis: object                  # torch float64 cuda, N*n^3 + n^2
    transform: np.ndarray          # (N, N) upper triangular
    collocation: np.ndarray        # (2N-1,) interleaved free-DoF indices
    solution_points: np.ndarray    # (N,)
    residual_points: np.ndarray    # (N-1,)
    chosen_mus: np.ndarray         # (N, p)
    indicator_history: np.ndarray
    saturated: bool = False
    chosen: np.ndarray | None = None
    layout: object = None            # FullNodeLayout for full-node problems (None: padded)
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def lay(self):
        return self.layout if self.layout is not None else PaddedLayout(self.n)

    @property
    def dim(self) -> int:
        return self.transform.shape[0]

    @property
    def n_points(self) -> int:
        return len(self.collocation)

    def basis_numpy(self) -> np.ndarray:
        """(n_free, N) basis in the reference's free-DoF ordering."""
        return self.lay.free_view(self.basis, self.dim).T.cpu().numpy()

    def prefix(self, N: int) -> "L1rocModel":
        if not 1 <= N <= self.dim:
            raise ValueError(f"prefix dimension {N} outside [1, {self.dim}]")
        lay = self.lay
        b = _vec(lay, N)
        b[: N * lay.S] = self.basis[: N * lay.S]
        return L1rocModel(self.n, b, self.transform[:N, :N].copy(), self.collocation[: 2 * N - 1],
                          self.solution_points[:N], self.residual_points[: N - 1],
                          self.chosen_mus[:N], self.indicator_history[:N], self.saturated,
                          None if self.chosen is None else self.chosen[:N], self.layout)

    # ---- device-side pieces of the online stage
    def _device(self, problem: ParametricProblem):
        import torch
        key = id(problem)
        if key in self._cache:
            return self._cache[key]
        n, N = self.n, self.dim
        lay = self.lay
        if layout_of(problem).side != n:
            raise ValueError("model and problem grids differ")
        rows = torch.as_tensor(lay.to_storage(self.collocation), device="cuda")
        M = len(self.collocation)
        Q = problem.spec.n_terms
        if lay.full_node:
            # full-node problems: A_q W from the batch-shared term coefficients with a unit
            # theta row per term (rbws_fn_apply_shared), then the collocation rows
            S, c = lay.S, problem.cells[-1]
            W = self.basis[: N * S].contiguous()
            parts = []
            for q in range(Q):
                th = torch.zeros(N, Q, dtype=torch.float64, device="cuda")
                th[:, q] = 1.0
                y = torch.empty(N * S, dtype=torch.float64, device="cuda")
                _native.call("rbws_fn_apply_shared", N, Q, c, th.data_ptr(),
                             problem._coef[-1].data_ptr(), W.data_ptr(), None, y.data_ptr(), 0,
                             _native.stream_ptr())
                parts.append(y.view(N, S)[:, rows].T)
            Bq = torch.stack(parts).contiguous().view(-1)
        elif getattr(problem, "stored", False):
            # assembled problems: per-term products A_q W from the stored coefficients,
            # then the collocation rows (the affine pieces of rb.py:200-201)
            n3 = n ** 3
            Bq = torch.stack([problem.term_apply(q, self.basis, N)[: N * n3].view(N, n3)[:, rows].T
                              for q in range(Q)]).contiguous().view(-1)
        else:
            Bq = torch.zeros(Q * M * N, dtype=torch.float64, device="cuda")
            _native.call("rbws_l1roc_project", problem.handle, self.basis.data_ptr(), n ** 3, N,
                         rows.data_ptr(), M, Bq.data_ptr(), _native.stream_ptr())
        T = torch.as_tensor(self.transform, dtype=torch.float64, device="cuda").contiguous()
        self._cache[key] = (rows, Bq, T)
        return self._cache[key]


def _online_batch(model: L1rocModel, problem, theta, f, count):
    """a, c, ind, status (device) for a batch; f padded rhs (shared or batch)."""
    import torch
    rows, Bq, T = model._device(problem)
    N, M, S = model.dim, len(model.collocation), model.lay.S
    f = f.reshape(-1)
    if f.numel() < count * S:  # one rhs shared by the batch
        bs = f[rows].contiguous()
        bstride = 0
    else:
        bs = f[: count * S].view(count, S)[:, rows].contiguous()
        bstride = M
    a = torch.empty(count * N, dtype=torch.float64, device="cuda")
    c = torch.empty(count * N, dtype=torch.float64, device="cuda")
    ind = torch.empty(count, dtype=torch.float64, device="cuda")
    st = torch.empty(count, dtype=torch.int32, device="cuda")
    _native.call("rbws_l1roc_online", count, problem.spec.n_terms, M, N, theta.data_ptr(),
                 Bq.data_ptr(), bs.data_ptr(), bstride, T.data_ptr(), a.data_ptr(),
                 c.data_ptr(), ind.data_ptr(), st.data_ptr(), _native.stream_ptr())
    return a, c, ind, st


def l1roc_online(model: L1rocModel, A, b, out=None, coords: bool = True):
    """Batched sub-sampled least-squares reduced solve (rb.py:190-205).

    A: BatchOperator (its context supplies theta(mu)); b: padded rhs.
    Returns (warm starts as a padded batch tensor, snapshot coordinates
    (count, N) numpy, or None with ``coords=False``).
    """
    import torch
    if model.dim == 0:
        raise ValueError("empty model")
    ctx = A.ctx
    problem, count = ctx.problem, ctx.count
    a, c, _, st = _online_batch(model, problem, ctx.theta, b, count)
    lay = model.lay
    n, S = lay.side, lay.S
    x = out if out is not None else _vec(lay, count)
    _native.call("rbws_expand", n, count, model.basis.data_ptr(), S, model.dim,
                 a.data_ptr(), x.data_ptr(), _native.stream_ptr())
    x[count * S:] = 0.0
    if lay.full_node:  # full-node batches are (count, nodes) tensors (fem_fn.py)
        x = x[: count * S].view(count, S)
    # one host sync, after the expansion is queued (x is discarded if the check fails)
    if np.any(_native.fetch(st) != 0):
        raise DegenerateBasisError("sub-sampled reduced system is rank deficient")
    return x, (_native.fetch(c.view(count, model.dim)) if coords else None)


# ----------------------------------------------------------------- DEIM

@dataclass
class DeimStep:
    column: object   # padded device vector (length n^3 + n^2)
    index: int       # free-DoF index (reference ordering)
    coeffs: np.ndarray
    pivot: float


def deim_extend(n: int, W, X, v, exclude=None) -> DeimStep:
    """Device DEIM extension (rb.py:96-126).

    W: padded tensor with len(X) columns (or None); X: free-DoF indices;
    v: padded single vector.  Returns the normalised column and new index.
    """
    import torch
    lay = n if hasattr(n, "side") else PaddedLayout(n)
    n, n3 = lay.side, lay.S
    v = v.reshape(-1)
    X = list(X)
    N = len(X)
    if N:
        pX = torch.as_tensor(lay.to_storage(X), device="cuda")
        Wm = W[: N * n3].view(N, n3)
        Aint = Wm[:, pX].T.contiguous()          # (N, N): W[X, :]
        bint = v[pX].contiguous()
        cvec = torch.empty(N, dtype=torch.float64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _native.call("rbws_dense_solve", N, Aint.data_ptr(), bint.data_ptr(), cvec.data_ptr(),
                     st.data_ptr(), _native.stream_ptr())
        if int(st.item()):
            raise DegenerateBasisError("singular DEIM interpolation matrix")
        wptr = W.data_ptr()
    else:
        cvec = torch.zeros(1, dtype=torch.float64, device="cuda")
        wptr = v.data_ptr()
    excl = torch.zeros(n3 + 2 * n * n, dtype=torch.uint8, device="cuda")
    if exclude:
        excl[torch.as_tensor(lay.to_storage(sorted(exclude)), device="cuda")] = 1
    col = torch.zeros(n3 + 2 * n * n, dtype=torch.float64, device="cuda")
    idx = torch.zeros(1, dtype=torch.int64, device="cuda")
    vals = torch.zeros(3, dtype=torch.float64, device="cuda")
    _native.call("rbws_deim_step_fn" if lay.full_node else "rbws_deim_step", n, wptr, n3, N,
                 cvec.data_ptr(), v.data_ptr(), excl.data_ptr(),
                 col.data_ptr(), idx.data_ptr(), vals.data_ptr(), _native.stream_ptr())
    pv, maxv, maxrho = (float(t) for t in vals.cpu())
    if maxrho <= 1e-14 * max(maxv, 1e-300):
        raise DegenerateBasisError("snapshot numerically inside the current basis")
    pidx = int(idx.item())
    if pidx < 0 or pv == 0.0:
        raise DegenerateBasisError("residual vanishes at all admissible points")
    index = int(lay.from_storage(pidx))
    return DeimStep(col, index, cvec[:N].cpu().numpy() if N else np.zeros(0), pv)


# ----------------------------------------------------------------- offline

def l1roc_offline(mus, N: int, hf_solve, problem: ParametricProblem, seed: int = 0,
                  progress=None, on_degenerate: str = "raise") -> L1rocModel:
    """Greedy offline training (rb.py:208-293) with device-side data work.

    on_degenerate: "raise" (reference behaviour, rb.py:116-117) or "stop" — end
    the greedy with the basis built so far (flagged as saturated) when a picked
    snapshot lies numerically inside the current basis.

    hf_solve(mu) -> padded device solution (e.g. hf.HighFidelitySolver).
    """
    import torch
    from .multigrid import mg_context_for
    mus = problem.spec.check_mus(mus)
    n_train = len(mus)
    if not 1 <= N <= n_train:
        raise ValueError("need 1 <= N <= number of training parameters")
    lay = layout_of(problem)
    n, n3 = lay.side, lay.S
    first = int(np.random.default_rng(seed).integers(n_train))
    # one rhs for every training parameter (assembled problems: mu-dependent data) or a
    # shared one
    per_mu = getattr(problem, "stored", False) or lay.full_node
    f = problem.rhs(mus).reshape(-1) if per_mu else problem.rhs()
    theta_train = problem.thetas(mus).contiguous()
    W = _vec(lay, N)
    R = _vec(lay, max(N - 1, 1))
    model_layout = lay if lay.full_node else None

    step = deim_extend(lay, None, [], hf_solve(mus[first]))
    W[:n3] = step.column[:n3]
    T = np.array([[step.pivot]])
    xs, xr, xi = [step.index], [], [step.index]
    chosen = [first]
    hist = [l1_indicator([1.0])]
    saturated = False
    ctx1 = None
    for nn in range(2, N + 1):
        taken = set(xs) | set(xr)
        cur = L1rocModel(n, W, T, np.asarray(xi, np.int64), np.asarray(xs, np.int64),
                         np.asarray(xr, np.int64), mus[chosen], np.asarray(hist),
                         layout=model_layout)
        a, c, ind, st = _online_batch(cur, problem, theta_train, f, n_train)
        if bool((st != 0).any()):
            raise DegenerateBasisError("sub-sampled reduced system is rank deficient")
        ind_h = ind.cpu().numpy()
        pick = int(np.argmax(ind_h))
        hist.append(float(ind_h[pick]))
        if progress:
            progress(f"greedy step {nn}: pick {pick} indicator {ind_h[pick]:.4g}")
        if pick in chosen:
            saturated = True
            break
        chosen.append(pick)
        u = hf_solve(mus[pick])
        m = nn - 1  # current basis width
        try:
            step = deim_extend(lay, W, xs, u, exclude=taken)
        except DegenerateBasisError:
            if on_degenerate != "stop":
                raise
            chosen.pop()
            saturated = True
            break
        taken.add(step.index)
        T = np.block([[T, step.coeffs[:, None]], [np.zeros((1, m)), np.array([[step.pivot]])]])
        W[m * n3:(m + 1) * n3] = step.column[:n3]
        xs.append(step.index)
        # residual snapshot r = f - A(mu_pick) (W[:, :m] a_pick)
        upick = _vec(lay, 1)
        apick = a[pick * m:(pick + 1) * m].contiguous()
        _native.call("rbws_expand", n, 1, W.data_ptr(), n3, m, apick.data_ptr(),
                     upick.data_ptr(), _native.stream_ptr())
        upick[n3:] = 0.0
        if lay.full_node:  # point-Jacobi context: operators only, no plane factorizations
            from .fem_fn import FnMgContext
            ctx1 = FnMgContext(problem, mus[pick][None], smoother="jacobi")
            Au = torch.zeros_like(upick)
            Au[:n3] = ctx1.apply(upick[:n3].view(1, n3)).view(-1)
        else:
            ctx1 = mg_context_for(problem, mus[pick][None], ctx=ctx1)
            Au = torch.zeros_like(upick)
            _native.call("rbws_apply", ctx1.handle, problem.finest_level, upick.data_ptr(),
                         Au.data_ptr(), _native.stream_ptr())
        fp = torch.zeros_like(upick)
        fp[:n3] = f[pick * n3:(pick + 1) * n3] if per_mu else f[:n3]
        r = fp - Au
        rstep = deim_extend(lay, R if xr else None, xr, r, exclude=taken)
        R[len(xr) * n3:(len(xr) + 1) * n3] = rstep.column[:n3]
        xr.append(rstep.index)
        xi.extend([step.index, rstep.index])
    Nf = len(xs)
    Wf = _vec(lay, Nf)
    Wf[: Nf * n3] = W[: Nf * n3]
    return L1rocModel(n, Wf, T, np.asarray(xi, np.int64), np.asarray(xs, np.int64),
                      np.asarray(xr, np.int64), mus[chosen], np.asarray(hist), saturated,
                      np.asarray(chosen, np.int64), model_layout)
