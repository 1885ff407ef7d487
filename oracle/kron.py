"""Matrix-free Kronecker-form oracle for large grids — TEST INFRASTRUCTURE ONLY.

At 256^3 and 512^3 the scipy route of ``oracle.problems`` (3D COO assembly of every
term, then Galerkin SpGEMM ``P^T A P`` per level, reference grid.py:173-182, 203-236)
needs tens of GB and many minutes per problem, so the large-size parity tests use this
restatement of the same operators instead:

* every affine term of the BASELINE problems is separable: the weight of the
  d-edge between nodes X and X + e_d is ``h * e_qd(X_d) * prod_{a != d} o_qa(X_a)``
  (the expressions of ``problems._face_weights``: exact block fractions, or the
  sin/sin/cos modes at the edge midpoint), so term q's free-free operator is
  ``sum_d Z_qd (x) Y_qd (x) X_qd`` (z slowest, x fastest, the reference's free-DoF
  order, problems.py:63-75) with a tridiagonal 1D stiffness on axis d and 1D
  diagonals on the other two;
* the free-DoF prolongation is ``P1 (x) P1 (x) P1`` (grid.py:131-141 restricted to
  interior nodes), so Galerkin coarsening acts factor by factor:
  ``P^T (Z (x) Y (x) X) P = (P1^T Z P1) (x) (P1^T Y P1) (x) (P1^T X P1)`` — exact
  in exact arithmetic, different only in rounding from the 3D SpGEMM;
* ``operator(mu, level)`` (grid.py:246-255) becomes a stencil: for every offset
  (a, b, c) in {-1, 0, 1}^3 a coefficient array
  ``C_abc[k, j, i] = sum_q theta_q sum_d Z_qd[k, k+c] Y_qd[j, j+b] X_qd[i, i+a]``;
  applying it is 7 (finest) or 27 (coarse) shifted multiply-adds;
* the V-cycle and PCG are the oracle's own (``solvers.mg_vcycle`` /
  ``solvers.mgcg_solve``, multigrid.py:205-232, krylov.py:42-109): the objects here
  duck-type ``A @ x``, ``A.diagonal()``, ``P @ e`` and ``P.T @ r``; the coarsest level
  is a dense matrix (Cholesky, multigrid.py:154-168).

``tests/test_oracle_kron.py`` checks this module against ``OracleProblem`` (3D
assembly) and the reference's golden V-cycle / MGCG vectors at small n.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import solvers as so
from .problems import FDProblemSpec, _overlap


# ---------------------------------------------------------------- 1D factors

def edge_node_factors(spec: FDProblemSpec, n: int, q: int, d: int):
    """1D factors of term q's d-edge weights on a grid with n cells.

    Returns ``(scale, fac)``: ``fac[a]`` for axis a is a length-(n+1) array; on axis d it
    is indexed by edge (edge i joins nodes i, i+1; entry n unused), on the other axes by
    node.  Edge weight = scale * prod_a fac[a][X_a] (problems._face_weights)."""
    h = 1.0 / n
    idx = np.arange(n + 1, dtype=np.float64)
    fac = []
    if spec.kind == "thermal-block":
        nb = spec.blocks
        a0, rem = q % nb[0], q // nb[0]
        cell = (a0, rem % nb[1], rem // nb[1])
        for ax in range(3):
            lo, hi = cell[ax] / nb[ax], (cell[ax] + 1) / nb[ax]
            if ax == d:
                mid = idx * h + 0.5 * h
                f = ((mid >= lo) & (mid < hi)).astype(np.float64)
            else:
                x = idx * h
                f = _overlap(x - 0.5 * h, x + 0.5 * h, lo, hi) / h
            fac.append(f)
        return h, fac
    for ax in range(3):
        x = idx * h + (0.5 * h if ax == d else 0.0)
        if q == 0:
            fac.append(np.ones(n + 1))
        else:
            fn = np.cos if ax == 2 else np.sin
            fac.append(fn(q * np.pi * x))
    return h, fac


def _stiffness(e: np.ndarray, c: int) -> sp.csr_matrix:
    """Interior block of the 1D edge Laplacian with edge weights e[0..c-1]."""
    e = e[:c]
    main = e[:-1] + e[1:]
    off = -e[1:-1]
    return sp.diags([off, main, off], [-1, 0, 1], shape=(c - 1, c - 1), format="csr")


def prolongation_1d(nc: int) -> sp.csr_matrix:
    """Interior rows/columns of the 1D linear interpolation nc -> 2nc (grid.py:131-141)."""
    nf = 2 * nc
    rows, cols, vals = [], [], []
    for s in range(1, nc):
        rows += [2 * s - 1, 2 * s, 2 * s + 1]
        cols += [s, s, s]
        vals += [0.5, 1.0, 0.5]
    P = sp.coo_matrix((vals, (np.asarray(rows) - 1, np.asarray(cols) - 1)),
                      shape=(nf - 1, nc - 1))
    return P.tocsr()


def _bands(M: sp.spmatrix) -> dict:
    """Tridiagonal matrix -> {offset: vector v with v[i] = M[i, i + offset]} (zeros outside)."""
    M = sp.csr_matrix(M)
    m = M.shape[0]
    out = {}
    for off in (-1, 0, 1):
        v = np.zeros(m)
        dg = M.diagonal(off)
        if off >= 0:
            v[:m - off] = dg
        else:
            v[-off:] = dg
        if np.any(v != 0.0):
            out[off] = v
    lo = sp.tril(M, -2).nnz + sp.triu(M, 2).nnz
    if lo:
        raise ValueError("factor is not tridiagonal")
    return out


class KronProblem:
    """Per-level Kronecker factors of every term (the ``OracleProblem`` operators)."""

    def __init__(self, spec: FDProblemSpec, n: int, m0: int = 4):
        if n % m0 or (n // m0) & (n // m0 - 1):
            raise ValueError("n must be m0 * 2^J")
        self.spec, self.n, self.m0 = spec, n, m0
        cells = [m0]
        while cells[-1] < n:
            cells.append(cells[-1] * 2)
        self.cells = tuple(cells)
        L = len(cells)
        # fac[l][q] = list over d of (Z, Y, X) 1D matrices (sparse), scale folded into X
        fine = []
        for q in range(spec.n_terms):
            per_d = []
            for d in range(3):
                scale, f = edge_node_factors(spec, n, q, d)
                mats = []
                for ax in range(3):
                    if ax == d:
                        mats.append(_stiffness(f[ax], n))
                    else:
                        mats.append(sp.diags(f[ax][1:n], 0, format="csr"))
                X, Y, Z = mats
                per_d.append((Z, Y, scale * X))
            fine.append(per_d)
        self.fac = [None] * L
        self.fac[-1] = fine
        self.P1 = [prolongation_1d(cells[i]) for i in range(L - 1)]
        for l in range(L - 2, -1, -1):
            P = self.P1[l]
            self.fac[l] = [[tuple((P.T @ M @ P).tocsr() for M in zyx) for zyx in per_d]
                           for per_d in self.fac[l + 1]]
        self.bands = [[[tuple(_bands(M) for M in zyx) for zyx in per_d] for per_d in lev]
                      for lev in self.fac]

    @property
    def levels(self) -> int:
        return len(self.cells)

    def rhs(self) -> np.ndarray:
        from .problems import rhs_full, interior_mask
        return rhs_full(self.spec, self.n)[~interior_mask(self.n)]

    def stencil(self, mu, level=None, k0=0, k1=None) -> "Stencil":
        """Coefficient arrays of operator(mu, level) for interior planes [k0, k1)."""
        if level is None:
            level = self.levels - 1
        m = self.cells[level] - 1
        k1 = m if k1 is None else k1
        th = self.spec.theta(mu)
        coef = {}
        for q, per_d in enumerate(self.bands[level]):
            for zb, yb, xb in per_d:
                for c, zv in zb.items():
                    zs = zv[k0:k1]
                    for b, yv in yb.items():
                        zy = th[q] * zs[:, None] * yv[None, :]
                        for a, xv in xb.items():
                            t = zy[:, :, None] * xv[None, None, :]
                            if (a, b, c) in coef:
                                coef[(a, b, c)] += t
                            else:
                                coef[(a, b, c)] = t
        return Stencil(m, k0, k1, coef)

    def dense(self, mu, level: int) -> np.ndarray:
        """Assembled operator of a (small) level as a dense matrix."""
        th = self.spec.theta(mu)
        A = None
        for q, per_d in enumerate(self.fac[level]):
            for Z, Y, X in per_d:
                t = th[q] * sp.kron(Z, sp.kron(Y, X))
                A = t if A is None else A + t
        return np.asarray(A.todense())

    def operator(self, mu, level=None):
        if level is None:
            level = self.levels - 1
        if level == 0:
            return self.dense(mu, 0)
        return self.stencil(mu, level)

    def prolongation(self, level: int) -> "KronProlongation":
        """Prolongation from level-1 to level."""
        return KronProlongation(self.P1[level - 1])


class Stencil:
    """operator(mu, level) on interior planes [k0, k1) as 7/27 coefficient arrays."""

    def __init__(self, m, k0, k1, coef):
        self.m, self.k0, self.k1, self.coef = m, k0, k1, coef
        self.shape = (m ** 3, m ** 3)

    def diagonal(self) -> np.ndarray:
        return self.coef[(0, 0, 0)].ravel().copy()

    def apply_planes(self, xpad: np.ndarray) -> np.ndarray:
        """xpad: (k1-k0+2, m+2, m+2) interior planes k0-1..k1 with a zero frame (planes
        outside [0, m) zero); returns (A x) on planes [k0, k1), shape (k1-k0, m, m)."""
        m, nz = self.m, self.k1 - self.k0
        y = np.zeros((nz, m, m))
        tmp = np.empty_like(y)
        for (a, b, c), C in self.coef.items():
            np.multiply(C, xpad[1 + c:1 + c + nz, 1 + b:1 + b + m, 1 + a:1 + a + m], out=tmp)
            y += tmp
        return y

    def __matmul__(self, x):
        m = self.m
        if self.k0 != 0 or self.k1 != m:
            raise ValueError("full-vector product needs the whole-level stencil")
        xp = np.zeros((m + 2, m + 2, m + 2))
        xp[1:-1, 1:-1, 1:-1] = np.asarray(x).reshape(m, m, m)
        return self.apply_planes(xp).ravel()


def _axis_apply(M: sp.spmatrix, X: np.ndarray, axis: int) -> np.ndarray:
    Xm = np.moveaxis(X, axis, 0)
    sh = Xm.shape
    Y = M @ Xm.reshape(sh[0], -1)
    return np.moveaxis(np.asarray(Y).reshape((M.shape[0],) + sh[1:]), 0, axis)


class KronProlongation:
    """P = P1 (x) P1 (x) P1 on interior DoFs; ``.T`` is the restriction P^T."""

    def __init__(self, P1: sp.spmatrix, transpose: bool = False):
        self.P1 = sp.csr_matrix(P1)
        self.transpose = transpose

    @property
    def T(self):
        return KronProlongation(self.P1, not self.transpose)

    def __matmul__(self, v):
        M = self.P1.T.tocsr() if self.transpose else self.P1
        mi = M.shape[1]
        X = np.asarray(v).reshape(mi, mi, mi)
        for ax in (2, 1, 0):
            X = _axis_apply(M, X, ax)
        return X.ravel()


def mg_context_for(kp: KronProblem, mu, nu: int = 1, omega: float = so.JACOBI_OMEGA):
    """The oracle's OracleMgContext (multigrid.py:191-202) on matrix-free operators."""
    ops = [kp.operator(mu, level=l) for l in range(kp.levels)]
    try:
        cf = sla.cho_factor(ops[0])
    except sla.LinAlgError as exc:
        raise so.OperatorError(f"coarsest operator not SPD: {exc}") from exc
    diags = [np.diag(ops[0]).copy()] + [A.diagonal() for A in ops[1:]]
    pros = [kp.prolongation(l) for l in range(1, kp.levels)]
    return so.OracleMgContext(ops, pros, diags, nu, cf, omega, "jacobi")


def mgcg_solve(kp: KronProblem, mu, delta=1e-10, l_max=60, x0=None):
    """Zero-init (or x0) MGCG on the matrix-free hierarchy (multigrid.py:225-232)."""
    ctx = mg_context_for(kp, mu)
    A = ctx.operators[-1]
    f = kp.rhs()
    x0 = np.zeros_like(f) if x0 is None else x0
    return so.mgcg_solve(A, f, x0, ctx, delta=delta, l_max=l_max, mu=mu)
