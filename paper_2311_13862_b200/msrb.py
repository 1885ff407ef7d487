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
* The online solve is ONE native call (rbws_msrbcg_solve, csrc/msrb.cu): the PCG loop with
  the iteration-indexed preconditioner, per-instance scalars and the active set on the
  device; this module only sets up the bases' reduced factors.
* Problems: the separable (Kronecker-factor) BASELINE problems and the reference's assembled
  Dirichlet problem example-1 (stored-coefficient hierarchy, per-parameter right-hand sides).

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
        Wr = W[:, rows]                                     # (N, M)
        if getattr(problem, "stored", False):
            # assembled problems: A_q W from the stored per-term coefficients
            AW = torch.stack([problem.term_apply(q, Wp, N)[: N * n ** 3].view(N, n ** 3)[:, rows]
                              for q in range(Q)])           # (Q, N, M), row b = A_q w_b
            self.red = torch.einsum("am,qbm->qab", Wr, AW).contiguous()
        else:
            Bq = torch.zeros(Q * m ** 3 * N, dtype=torch.float64, device="cuda")
            _native.call("rbws_l1roc_project", problem.handle, Wp.data_ptr(), n ** 3, N,
                         rows.data_ptr(), m ** 3, Bq.data_ptr(), _native.stream_ptr())
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


def _padded_only(problem):
    """rbi-msrbcg runs on the padded interior layout: the separable BASELINE problems and
    assembled Dirichlet problems (example-1).  Full-node problems (example-2: free boundary
    nodes) have no Gauss-Seidel sweep on that layout."""
    if hasattr(problem, "masks"):
        raise NotImplementedError(f"{problem.spec.pid}: rbi-msrbcg needs the symmetric "
                                  "Gauss-Seidel sweep, which the full-node layout does not have; "
                                  "use mgcg / rbi-mgcg")


def _rhs_rows(problem, mus, f=None):
    """(count, n^3) right-hand sides: per parameter for assembled problems (lifted Dirichlet
    data, grid.py:266-284), one shared vector expanded for the separable ones."""
    cnt, n3 = len(mus), problem.n ** 3
    if f is None:
        f = problem.rhs(mus) if getattr(problem, "stored", False) else problem.rhs()
    f = f.reshape(-1)
    if f.numel() >= cnt * n3 and (cnt > 1 or getattr(problem, "stored", False)):
        return f[: cnt * n3].view(cnt, n3)
    return f[:n3].view(1, n3).expand(cnt, n3)


def msrb_train(mus, N: int, K_max: int, hf_solver, problem) -> MsrbHierarchy:
    """Per-iteration error-snapshot bases (msrb.py:113-149); hf_solver: HighFidelitySolver."""
    _padded_only(problem)
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
    f = _rhs_rows(problem, mus)
    red0 = _Reduced(problem, init.basis)
    x = red0.solve(red0.factor(theta), f.contiguous()) if red0.N else \
        torch.zeros(cnt, n3, dtype=torch.float64, device="cuda")
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
    (msrb.py:53-85) as one native call (rbws_msrbcg_solve).  Returns (x padded device
    vector, SolveReports)."""
    _padded_only(problem)
    import ctypes

    import torch
    from .multigrid import mg_context_for
    if delta <= 0:
        raise ValueError("tolerance must be positive")
    if l_max < 0:
        raise ValueError("l_max must be non-negative")
    mus = problem.spec.check_mus(mus)
    cnt, n, n3 = len(mus), problem.n, problem.n ** 3
    if ctx is None or ctx.smoother_kind != "gs" or ctx.count != cnt:
        ctx = mg_context_for(problem, mus, smoother="gs", ctx=ctx)
    theta = ctx.theta
    frows = _rhs_rows(problem, mus, f)
    shared = frows.stride(0) == 0
    fbuf = torch.zeros(padded_len(n, 1 if shared else cnt), dtype=torch.float64, device="cuda")
    fbuf[: (1 if shared else cnt) * n3] = (frows[0] if shared else frows).reshape(-1)
    t0 = time.perf_counter()
    # the POD Galerkin initial guess and the reduced factors of every iteration's basis
    red0 = _Reduced(problem, hier.init_basis.basis)
    xp = torch.zeros(padded_len(n, cnt), dtype=torch.float64, device="cuda")
    if red0.N:
        xp[: cnt * n3] = red0.solve(red0.factor(theta), frows.contiguous()).reshape(-1)
    keep, Ws, strides, Ns, chols = [], [], [], [], []
    for W in hier.bases:
        Wc = W.contiguous()
        red = _Reduced(problem, Wc)
        Lk = red.factor(theta).contiguous() if red.N else None
        keep.append((Wc, Lk))
        Ws.append(Wc.data_ptr() if red.N else 0)
        strides.append(Wc.stride(0) if red.N else 0)
        Ns.append(red.N)
        chols.append(Lk.data_ptr() if red.N else 0)
    nb = len(Ws)
    Wa = (ctypes.c_void_p * max(nb, 1))(*Ws)
    Sa = (ctypes.c_int64 * max(nb, 1))(*strides)
    Na = (ctypes.c_int * max(nb, 1))(*Ns)
    Ca = (ctypes.c_void_p * max(nb, 1))(*chols)
    iters = np.zeros(cnt, dtype=np.int32)
    hist = np.zeros((cnt, l_max + 1))
    tres = np.zeros(cnt)
    status = np.zeros(cnt, dtype=np.int32)
    _native.call("rbws_msrbcg_solve", ctx.handle, fbuf.data_ptr(), 0 if shared else n3,
                 xp.data_ptr(), float(delta), int(l_max), nb, Wa, Sa, Na, Ca, iters.ctypes.data,
                 hist.ctypes.data, tres.ctypes.data, status.ctypes.data, _native.stream_ptr())
    torch.cuda.current_stream().synchronize()
    del keep
    if np.any(status & 1):
        raise OperatorError("non-positive curvature p.A.p; operator not SPD")
    reps = SolveReports(method, iters, hist, tres, status, time.perf_counter() - t0, delta, l_max,
                        mus, {"batch": cnt, "smoother": "gauss-seidel-symmetric",
                              "K_max": hier.K_max, "N": hier.N})
    return xp, reps
