"""CPU oracle (test infrastructure only) of the reference's multispace reduced-basis
preconditioner and the rbi-msrbcg method (reference msrb.py, rb.py:45-86,
warmstart.py:70-117).  Restatement with numpy/scipy; pinned against golden vectors of the
real reference (tests/golden/make_golden.py --msrb).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from .solvers import gs_sweep, pcg_solve


@dataclass
class PodBasis:
    """Orthonormal basis from the method of snapshots (rb.py:33-42)."""

    basis: np.ndarray
    eigenvalues: np.ndarray
    n_snapshots: int


def pod_build(snapshots, N: int) -> PodBasis:
    """Correlation-matrix eigendecomposition, truncation at rank 1e-14, QR with sign fix
    (rb.py:45-68)."""
    S = np.column_stack([np.asarray(s, dtype=np.float64) for s in snapshots])
    n_s = S.shape[1]
    w, V = np.linalg.eigh(S.T @ S)
    w = w[::-1].copy()
    V = V[:, ::-1]
    w[w < 0.0] = 0.0
    rank = int(np.sum(w > 1e-14 * max(w[0], 1e-300)))
    N_eff = min(N, rank)
    if N_eff == 0:
        return PodBasis(np.zeros((S.shape[0], 0)), w, n_s)
    W = S @ (V[:, :N_eff] / np.sqrt(w[:N_eff]))
    Q, R = np.linalg.qr(W)
    return PodBasis(Q * np.sign(np.diag(R)), w, n_s)


def rbm_pod_solve(A, b, W) -> np.ndarray:
    """Galerkin reduced solve W (W^T A W)^{-1} W^T b (rb.py:71-86)."""
    W = np.asarray(W)
    if W.shape[1] == 0:
        return np.zeros(W.shape[0])
    return W @ sla.solve(W.T @ (A @ W), W.T @ np.asarray(b, dtype=np.float64), assume_a="sym")


def sgs_sweep(A, b) -> np.ndarray:
    """One symmetric Gauss-Seidel sweep from zero (FINE_SMOOTH, msrb.py:20, kernels.py:93-95)."""
    x = np.zeros(A.shape[0])
    gs_sweep(A, x, b, True)
    gs_sweep(A, x, b, False)
    return x


def msrb_apply(b, A, W) -> np.ndarray:
    """One smoothing sweep plus the reduced correction of its residual (msrb.py:40-50)."""
    u = sgs_sweep(A, b)
    if W.shape[1] == 0:
        return u
    return u + rbm_pod_solve(A, b - A @ u, W)


@dataclass
class MsrbHierarchy:
    init_basis: PodBasis
    bases: tuple
    N: int
    K_max: int

    def basis_for(self, k: int) -> np.ndarray:
        if not self.bases:
            return np.zeros((self.init_basis.basis.shape[0], 0))
        return self.bases[min(k, len(self.bases) - 1)]


def msrb_train(mus, N: int, K_max: int, hf_solver, operator, rhs) -> MsrbHierarchy:
    """Per-iteration error-snapshot bases from the simulated reduced-initialised,
    MSRB-preconditioned CG over the training set (msrb.py:113-149)."""
    mus = [np.asarray(m, dtype=np.float64) for m in mus]
    init = pod_build([hf_solver(m) for m in mus], N)
    if K_max == 0:
        return MsrbHierarchy(init, (), N, 0)
    systems = [(operator(m), rhs(m)) for m in mus]
    states = []
    for A, f in systems:
        x = rbm_pod_solve(A, f, init.basis)
        states.append({"x": x, "r": f - A @ x, "p": None, "rs": None})
    bases = []
    for _k in range(K_max):
        pod_k = pod_build([hf_solver(m, st["r"]) for m, st in zip(mus, states)], N)
        bases.append(pod_k.basis)
        for (A, _f), st in zip(systems, states):   # _PcgState.advance (msrb.py:88-110)
            s = msrb_apply(st["r"], A, pod_k.basis)
            rs_new = float(st["r"] @ s)
            st["p"] = s if st["p"] is None else s + (rs_new / st["rs"]) * st["p"]
            st["rs"] = rs_new
            Ap = A @ st["p"]
            alpha = st["rs"] / float(st["p"] @ Ap)
            st["x"] = st["x"] + alpha * st["p"]
            st["r"] = st["r"] - alpha * Ap
    return MsrbHierarchy(init, tuple(bases), N, K_max)


def rbi_msrbcg_solve(A, f, hier: MsrbHierarchy, delta=1e-10, l_max=40):
    """rbi-msrbcg: POD Galerkin initial guess, PCG with the iteration-indexed MSRB
    preconditioner (warmstart.py:81-117, msrb.py:53-85)."""
    u0 = rbm_pod_solve(A, f, hier.init_basis.basis)
    return pcg_solve(A, f, u0, precond=lambda r, k: msrb_apply(r, A, hier.basis_for(k)),
                     delta=delta, l_max=l_max, method="rbi-msrbcg")
