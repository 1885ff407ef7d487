"""Multispace reduced-basis preconditioning on the B200 (reference msrb.py, rb.py:33-86).

rbi-msrbcg = POD Galerkin initial guess + PCG whose k-th preconditioner is one symmetric
Gauss-Seidel sweep from zero plus a Galerkin correction of its residual in the k-th
error-snapshot POD space.  Batched over parameters:

* POD (rb.py:45-68): the snapshot correlation S^T S and the lift S V are FP64 library
  GEMMs on the device (cuBLAS through torch), the small symmetric eigenproblem on the host;
  QR with the reference's sign convention.
* Reduced operators: W^T A_q W per affine term, from the native per-term products
  (rbws_l1roc_project over all interior rows) — the "V^T (A_q V)" projection, N <= a few
  tens of columns: a skinny FP64 product done once per basis; per parameter the reduced
  matrix is sum_q theta_q W^T A_q W and its Cholesky factor is batched.
* Sweeps and residuals are the native kernels (rbws_smooth symmetric Gauss-Seidel,
  rbws_level_kernel residual, rbws_apply).

Semantics follow the reference: msrb_train simulates the reduced-initialised,
MSRB-preconditioned CG over the training set, one iteration per basis index
(msrb.py:113-149); the preconditioner for iteration k >= K_max reuses the last basis.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .grid import interior_to_padded_index, padded_len
from .krylov import OperatorError, SolveReports
from .multigrid import MgContext


@dataclass
class PodBasis:
    """Orthonormal basis (N padded device vectors) from the method of snapshots."""

    basis: object        # torch (N, n^3) float64, padded layout rows
    eigenvalues: np.ndarray
    n_snapshots: int

    @property
    def dim(self) -> int:
        return int(self.basis.shape[0])


def pod_build(S, N: int) -> PodBasis:
    """POD of the snapshot rows S (torch (n_s, n^3), padded vectors): rb.py:45-68."""
    import torch
    n_s = S.shape[0]
    C = (S @ S.T).cpu().numpy()
    w, V = np.linalg.eigh(C)
    w = w[::-1].copy()
    V = V[:, ::-1]
    w[w < 0.0] = 0.0
    rank = int(np.sum(w > 1e-14 * max(w[0], 1e-300)))
    N_eff = min(N, rank)
    if N_eff == 0:
        return PodBasis(S.new_zeros((0, S.shape[1])), w, n_s)
    coef = torch.as_tensor(np.ascontiguousarray(V[:, :N_eff] / np.sqrt(w[:N_eff])),
                           dtype=torch.float64, device=S.device)
    Wt = S.T @ coef                       # (n^3, N)
    Q, R = torch.linalg.qr(Wt)
    Q = Q * torch.sign(torch.diagonal(R))[None, :]
    return PodBasis(Q.T.contiguous(), w, n_s)


class _Reduced:
    """W^T A_q W for every affine term of one basis (the skinny projection)."""

    def __init__(self, problem, W):
        import torch
        n, N, Q = problem.n, int(W.shape[0]), problem.spec.n_terms
        self.W, self.N, self.n = W, N, n
        if N == 0:
            self.red = None
            return
        m = n - 1
        rows = torch.as_tensor(interior_to_padded_index(np.arange(m ** 3), n), device="cuda")
        Wp = torch.zeros(padded_len(n, N), dtype=torch.float64, device="cuda")
        Wp[: N * n ** 3] = W.reshape(-1)
        Bq = torch.zeros(Q * m ** 3 * N, dtype=torch.float64, device="cuda")
        _native.call("rbws_l1roc_project", problem.handle, Wp.data_ptr(), n ** 3, N,
                     rows.data_ptr(), m ** 3, Bq.data_ptr(), _native.stream_ptr())
        Wr = W[:, rows]                                     # (N, M)
        self.red = torch.einsum("am,qmb->qab", Wr, Bq.view(Q, m ** 3, N)).contiguous()

    def factor(self, theta):
        """Cholesky factors of sum_q theta_q W^T A_q W for a batch (count, Q)."""
        import torch
        A_N = torch.einsum("cq,qab->cab", theta, self.red)
        A_N = 0.5 * (A_N + A_N.transpose(1, 2))
        L, info = torch.linalg.cholesky_ex(A_N)
        if bool((info != 0).any()):
            from .rb import DegenerateBasisError
            raise DegenerateBasisError("reduced operator not SPD")
        return L

    def solve(self, L, b):
        """W (A_N)^{-1} W^T b for every instance row of b (count, n^3): the projections
        W^T b (rbws_basis_dot) and the expansion W t (rbws_expand) are the library's
        memory-bound kernels; the N x N Cholesky solves are per-instance torch calls."""
        import torch
        count, n3 = b.shape
        N = self.N
        Wc = self.W.contiguous()
        t = torch.empty(count, N, dtype=torch.float64, device="cuda")
        st = _native.stream_ptr()
        _native.call("rbws_basis_dot", n3, count, Wc.data_ptr(), Wc.stride(0), N, b.data_ptr(),
                     b.stride(0), t.data_ptr(), st)
        t = torch.cholesky_solve(t.unsqueeze(-1), L).squeeze(-1).contiguous()
        out = torch.empty(count * n3 + 2 * self.n * self.n, dtype=torch.float64, device="cuda")
        _native.call("rbws_expand", self.n, count, Wc.data_ptr(), Wc.stride(0), N, t.data_ptr(),
                     out.data_ptr(), st)
        return out[: count * n3].view(count, n3)


@dataclass
class MsrbHierarchy:
    """Initial POD space plus one error-snapshot basis per iteration index (msrb.py:23-37)."""

    init_basis: PodBasis
    bases: tuple
    N: int
    K_max: int
    spectra: tuple = ()

    def basis_for(self, k: int):
        return self.bases[min(k, len(self.bases) - 1)] if self.bases else None


class _BatchOps:
    """Native operator / sweep / residual for one MgContext batch on (count, n^3) views."""

    def __init__(self, ctx: MgContext):
        import torch
        self.ctx, n = ctx, ctx.problem.n
        self.n3, self.L = n ** 3, ctx.problem.levels - 1
        self.count = ctx.count
        self._buf = [torch.zeros(padded_len(n, ctx.count), dtype=torch.float64, device="cuda")
                     for _ in range(3)]

    def _pad(self, i, v):
        b = self._buf[i]
        b[: self.count * self.n3] = v.reshape(-1)
        return b

    def apply(self, v):
        y = self._buf[2]
        _native.call("rbws_apply", self.ctx.handle, self.L, self._pad(0, v).data_ptr(),
                     y.data_ptr(), _native.stream_ptr())
        return y[: self.count * self.n3].view(self.count, self.n3).clone()

    def sgs(self, r):
        """One symmetric Gauss-Seidel sweep from zero on rhs r (FINE_SMOOTH)."""
        x = self._buf[1]
        x.zero_()
        _native.call("rbws_smooth", self.ctx.handle, self.L, 3, x.data_ptr(),
                     self._pad(0, r).data_ptr(), _native.stream_ptr())
        return x[: self.count * self.n3].view(self.count, self.n3).clone()


def _apply_precond(ops, red: _Reduced | None, L, r):
    u = ops.sgs(r)
    if red is None or red.N == 0:
        return u
    return u + red.solve(L, r - ops.apply(u))


def _separable_only(problem):
    if getattr(problem, "stored", False):
        raise NotImplementedError("rbi-msrbcg runs on the separable (Kronecker-factor) problems; "
                                  "assembled problems take mgcg / rbi-mgcg")


def msrb_train(mus, N: int, K_max: int, hf_solver, problem) -> MsrbHierarchy:
    """Per-iteration error-snapshot bases (msrb.py:113-149); hf_solver: HighFidelitySolver."""
    _separable_only(problem)
    import torch
    if K_max < 0:
        raise ValueError("K_max must be non-negative")
    mus = problem.spec.check_mus(mus)
    n3, cnt = problem.n ** 3, len(mus)
    snaps = hf_solver.solve_batch(mus)[: cnt * n3].view(cnt, n3).clone()
    init = pod_build(snaps, N)
    if K_max == 0:
        return MsrbHierarchy(init, (), N, 0)
    from .multigrid import mg_context_for
    ctx = mg_context_for(problem, mus, smoother="gs")
    ops = _BatchOps(ctx)
    theta = ctx.theta
    f = problem.rhs()[:n3].view(1, n3).expand(cnt, n3)
    red0 = _Reduced(problem, init.basis)
    x = red0.solve(red0.factor(theta), f) if red0.N else torch.zeros(cnt, n3, dtype=torch.float64,
                                                                       device="cuda")
    r = f - ops.apply(x)
    p, rs = None, None
    bases, spectra = [], []
    for _k in range(K_max):
        rp = torch.zeros(padded_len(problem.n, cnt), dtype=torch.float64, device="cuda")
        rp[: cnt * n3] = r.reshape(-1)
        errs = hf_solver.solve_batch(mus, rhs=rp)[: cnt * n3].view(cnt, n3).clone()
        pod_k = pod_build(errs, N)
        bases.append(pod_k.basis)
        spectra.append(pod_k.eigenvalues)
        red = _Reduced(problem, pod_k.basis)
        s = _apply_precond(ops, red, red.factor(theta) if red.N else None, r)
        rs_new = (r * s).sum(1)                      # _PcgState.advance (msrb.py:88-110)
        p = s if p is None else s + (rs_new / rs)[:, None] * p
        rs = rs_new
        Ap = ops.apply(p)
        alpha = rs / (p * Ap).sum(1)
        x = x + alpha[:, None] * p
        r = r - alpha[:, None] * Ap
    return MsrbHierarchy(init, tuple(bases), N, K_max, tuple(spectra))


def rbi_msrbcg_solve(problem, mus, hier: MsrbHierarchy, f=None, delta: float = 1e-16,
                     l_max: int = 40, method: str = "rbi-msrbcg", ctx: MgContext | None = None):
    """Batched rbi-msrbcg: POD Galerkin initial guess (warmstart.py:81-84), then PCG
    (krylov.py:42-109 semantics, per instance) with the MSRB preconditioner
    (msrb.py:53-85).  Returns (x (count, n^3) padded rows, SolveReports)."""
    _separable_only(problem)
    import torch
    from .multigrid import mg_context_for
    mus = problem.spec.check_mus(mus)
    cnt, n3 = len(mus), problem.n ** 3
    if ctx is None or ctx.smoother_kind != "gs" or ctx.count != cnt:
        ctx = mg_context_for(problem, mus, smoother="gs", ctx=ctx)
    ops = _BatchOps(ctx)
    theta = ctx.theta
    f = (problem.rhs() if f is None else f)[:n3].view(1, n3).expand(cnt, n3)
    t0 = time.perf_counter()
    red_cache = {}

    def reduced(k):
        W = hier.basis_for(k)
        key = -1 if W is None else min(k, len(hier.bases) - 1)
        if key not in red_cache:
            red = None if W is None else _Reduced(problem, W)
            red_cache[key] = (red, red.factor(theta) if red is not None and red.N else None)
        return red_cache[key]

    red0 = _Reduced(problem, hier.init_basis.basis)
    x = red0.solve(red0.factor(theta), f) if red0.N else torch.zeros(cnt, n3, dtype=torch.float64,
                                                                       device="cuda")
    fn = torch.linalg.vector_norm(f, dim=1)
    absolute = (fn == 0)
    scale = torch.where(absolute, torch.ones_like(fn), fn)
    r = f - ops.apply(x)
    rel = torch.linalg.vector_norm(r, dim=1) / scale
    hist = [rel]  # device tensors, copied to the host once at the end
    iters_d = torch.zeros(cnt, dtype=torch.int32, device="cuda")
    active = (rel > delta) if l_max > 0 else torch.zeros_like(rel, dtype=torch.bool)
    status = np.zeros(cnt, dtype=np.int32)
    if bool(active.any()):
        red, L = reduced(0)
        s = _apply_precond(ops, red, L, r)
        p = s
        rs = (r * s).sum(1)
        k = 0
        while k < l_max and bool(active.any()):
            Ap = ops.apply(p)
            pAp = (p * Ap).sum(1)
            bad = active & ~(pAp > 0)
            if bool(bad.any()):
                raise OperatorError("non-positive curvature p.A.p; operator not SPD")
            alpha = torch.where(active, rs / pAp, torch.zeros_like(rs))
            x = x + alpha[:, None] * p
            r = r - alpha[:, None] * Ap
            k += 1
            rel_k = torch.linalg.vector_norm(r, dim=1) / scale
            iters_d = torch.where(active, torch.full_like(iters_d, k), iters_d)
            hist.append(torch.where(active, rel_k, torch.full_like(rel_k, float("nan"))))
            active = active & (rel_k > delta)
            if not bool(active.any()) or k >= l_max:
                break
            red, L = reduced(k)
            s = _apply_precond(ops, red, L, r)
            rs_new = (r * s).sum(1)
            p = s + (rs_new / rs)[:, None] * p
            rs = rs_new
    tres = (torch.linalg.vector_norm(f - ops.apply(x), dim=1) / scale).cpu().numpy()
    status |= np.where(absolute.cpu().numpy(), 4, 0).astype(np.int32)
    iters = iters_d.cpu().numpy()
    H = np.full((cnt, l_max + 1), np.nan)
    Hd = torch.stack(hist, 1).cpu().numpy()
    H[:, : Hd.shape[1]] = Hd
    reps = SolveReports(method, iters, H, tres, status, time.perf_counter() - t0, delta, l_max,
                        mus, {"batch": cnt, "smoother": "gauss-seidel-symmetric",
                              "K_max": hier.K_max, "N": hier.N})
    xp = torch.zeros(padded_len(problem.n, cnt), dtype=torch.float64, device="cuda")
    xp[: cnt * n3] = x.reshape(-1)
    return xp, reps
