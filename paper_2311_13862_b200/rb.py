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
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def dim(self) -> int:
        return self.transform.shape[0]

    @property
    def n_points(self) -> int:
        return len(self.collocation)

    def basis_numpy(self) -> np.ndarray:
        """(n_free, N) basis in the reference's free-DoF ordering."""
        n, N = self.n, self.dim
        blk = self.basis[: N * n ** 3].view(N, n, n, n)[:, 1:, 1:, 1:]
        return blk.reshape(N, -1).T.cpu().numpy()

    def prefix(self, N: int) -> "L1rocModel":
        if not 1 <= N <= self.dim:
            raise ValueError(f"prefix dimension {N} outside [1, {self.dim}]")
        n = self.n
        import torch
        b = torch.zeros(padded_len(n, N), dtype=torch.float64, device="cuda")
        b[: N * n ** 3] = self.basis[: N * n ** 3]
        return L1rocModel(n, b, self.transform[:N, :N].copy(), self.collocation[: 2 * N - 1],
                          self.solution_points[:N], self.residual_points[: N - 1],
                          self.chosen_mus[:N], self.indicator_history[:N], self.saturated,
                          None if self.chosen is None else self.chosen[:N])

    # ---- device-side pieces of the online stage
    def _device(self, problem: ParametricProblem):
        import torch
        key = id(problem)
        if key in self._cache:
            return self._cache[key]
        n, N = self.n, self.dim
        if problem.n != n:
            raise ValueError("model and problem grids differ")
        rows = torch.as_tensor(interior_to_padded_index(self.collocation, n), device="cuda")
        M = len(self.collocation)
        Q = problem.spec.n_terms
        if getattr(problem, "stored", False):
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
    n, N, M = model.n, model.dim, len(model.collocation)
    if f.numel() == padded_len(n, 1):
        bs = f[rows].contiguous()
        bstride = 0
    else:
        bs = f[: count * n ** 3].view(count, n ** 3)[:, rows].contiguous()
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
    n = model.n
    x = out if out is not None else torch.empty(padded_len(n, count), dtype=torch.float64,
                                                device="cuda")
    _native.call("rbws_expand", n, count, model.basis.data_ptr(), n ** 3, model.dim,
                 a.data_ptr(), x.data_ptr(), _native.stream_ptr())
    x[count * n ** 3:] = 0.0
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
    X = list(X)
    N = len(X)
    n3 = n ** 3
    if N:
        pX = torch.as_tensor(interior_to_padded_index(X, n), device="cuda")
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
    excl = torch.zeros(padded_len(n, 1), dtype=torch.uint8, device="cuda")
    if exclude:
        excl[torch.as_tensor(interior_to_padded_index(sorted(exclude), n), device="cuda")] = 1
    col = torch.zeros(padded_len(n, 1), dtype=torch.float64, device="cuda")
    idx = torch.zeros(1, dtype=torch.int64, device="cuda")
    vals = torch.zeros(3, dtype=torch.float64, device="cuda")
    _native.call("rbws_deim_step", n, wptr, n3, N, cvec.data_ptr(), v.data_ptr(), excl.data_ptr(),
                 col.data_ptr(), idx.data_ptr(), vals.data_ptr(), _native.stream_ptr())
    pv, maxv, maxrho = (float(t) for t in vals.cpu())
    if maxrho <= 1e-14 * max(maxv, 1e-300):
        raise DegenerateBasisError("snapshot numerically inside the current basis")
    pidx = int(idx.item())
    if pidx < 0 or pv == 0.0:
        raise DegenerateBasisError("residual vanishes at all admissible points")
    index = int(padded_to_interior_index(pidx, n))
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
    n = problem.n
    n3 = n ** 3
    first = int(np.random.default_rng(seed).integers(n_train))
    # one rhs for every training parameter (assembled problems: mu-dependent data) or a
    # shared one
    stored = getattr(problem, "stored", False)
    f = problem.rhs(mus) if stored else problem.rhs()
    theta_train = problem.thetas(mus).contiguous()
    W = torch.zeros(padded_len(n, N), dtype=torch.float64, device="cuda")
    R = torch.zeros(padded_len(n, max(N - 1, 1)), dtype=torch.float64, device="cuda")

    step = deim_extend(n, None, [], hf_solve(mus[first]))
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
                         np.asarray(xr, np.int64), mus[chosen], np.asarray(hist))
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
            step = deim_extend(n, W, xs, u, exclude=taken)
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
        ctx1 = mg_context_for(problem, mus[pick][None], ctx=ctx1)
        upick = torch.zeros(padded_len(n, 1), dtype=torch.float64, device="cuda")
        apick = a[pick * m:(pick + 1) * m].contiguous()
        _native.call("rbws_expand", n, 1, W.data_ptr(), n3, m, apick.data_ptr(),
                     upick.data_ptr(), _native.stream_ptr())
        upick[n3:] = 0.0
        Au = torch.zeros_like(upick)
        _native.call("rbws_apply", ctx1.handle, problem.finest_level, upick.data_ptr(),
                     Au.data_ptr(), _native.stream_ptr())
        fp = f[pick * n3:(pick + 1) * n3 + 2 * n * n] if stored else f
        r = fp - Au
        rstep = deim_extend(n, R if xr else None, xr, r, exclude=taken)
        R[len(xr) * n3:(len(xr) + 1) * n3] = rstep.column[:n3]
        xr.append(rstep.index)
        xi.extend([step.index, rstep.index])
    Nf = len(xs)
    Wf = torch.zeros(padded_len(n, Nf), dtype=torch.float64, device="cuda")
    Wf[: Nf * n3] = W[: Nf * n3]
    return L1rocModel(n, Wf, T, np.asarray(xi, np.int64), np.asarray(xs, np.int64),
                      np.asarray(xr, np.int64), mus[chosen], np.asarray(hist), saturated,
                      np.asarray(chosen, np.int64))
