"""Oracle problem definitions and per-level affine operators — TEST INFRASTRUCTURE ONLY.

The BASELINE configurations are finite-volume (7-point, vertex-centred)
discretisations of -div(a(x; mu) grad u) = f on the unit cube with
homogeneous Dirichlet data.  The reference package only ships trilinear-FEM
assembly; its solver stack (Galerkin coarsening, smoothers, PCG, L1ROC) is
discretisation-agnostic, so these operators are fed to it through the same
``ParametricProblem`` interface (reference grid.py:193-290) and the golden
script injects them into the reference unchanged.

Discretisation (documented in DESIGN.md §2):

* grid: n cells per axis, nodes (n+1)^3, free DoFs = interior nodes in
  lexicographic x-fastest order (reference problems.py:63-75, grid.py:205-210);
* operator of affine term q: sum over grid edges of
  ``w_q(edge) * (u_X - u_Y)^2 / 2`` where the edge weight is ``h`` times the
  mean of the term's coefficient over the dual face (an h x h square centred at
  the edge midpoint, normal to the edge).  Thermal blocks: exact face fractions;
  smooth affine coefficient: midpoint rule;
* rhs: ``h^3 f(X)`` at interior nodes.

This module assembles every term directly in 3D with scipy (no separable
shortcut), so it is an independent check of the product's Kronecker-factored
tables.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass(frozen=True)
class FDProblemSpec:
    """A parametrised FV diffusion problem (mirrors reference problems.py:26-53)."""

    pid: str
    kind: str                      # "thermal-block" | "smooth-affine"
    p: int                         # parameter dimension
    bounds: tuple                  # ((lo, hi),) * p
    blocks: tuple = (1, 1, 1)      # thermal block counts (bx, by, bz)
    sampling: str = "log-uniform"  # how BASELINE draws mu
    n_modes: int = 0               # smooth-affine modes

    @property
    def n_terms(self) -> int:
        return self.p if self.kind == "thermal-block" else self.n_modes + 1

    def theta(self, mu) -> np.ndarray:
        """Affine weights theta_q(mu) (reference problems.py:18-23 DiffusionTerm.theta)."""
        mu = self.check_mu(mu)
        if self.kind == "thermal-block":
            return mu.copy()
        return np.concatenate([[1.0], mu])

    def check_mu(self, mu) -> np.ndarray:
        """Shape/bounds validation, as reference problems.py:47-53."""
        mu = np.asarray(mu, dtype=np.float64)
        if mu.shape != (self.p,):
            raise ValueError(f"{self.pid} expects {self.p}-dimensional parameters")
        b = np.asarray(self.bounds, dtype=np.float64)
        if np.any(mu < b[:, 0]) or np.any(mu > b[:, 1]):
            raise ValueError(f"parameter {mu} outside {self.pid} bounds")
        return mu


def thermal_block(blocks=(2, 1, 1)) -> FDProblemSpec:
    bx, by, bz = blocks
    p = bx * by * bz
    return FDProblemSpec(pid=f"thermal-block-{bx}x{by}x{bz}", kind="thermal-block",
                         p=p, bounds=((0.1, 10.0),) * p, blocks=(bx, by, bz),
                         sampling="log-uniform")


def smooth_affine(n_modes: int = 6) -> FDProblemSpec:
    return FDProblemSpec(pid=f"smooth-affine-{n_modes}", kind="smooth-affine",
                         p=n_modes, bounds=((-0.1, 0.1),) * n_modes,
                         sampling="uniform", n_modes=n_modes)


def sample_mus(spec: FDProblemSpec, count: int, seed: int) -> np.ndarray:
    """BASELINE.json sampling: log-uniform in [0.1,10]^p or uniform in the box."""
    rng = np.random.default_rng(seed)
    b = np.asarray(spec.bounds, dtype=np.float64)
    u = rng.random((count, spec.p))
    if spec.sampling == "log-uniform":
        lo, hi = np.log(b[:, 0]), np.log(b[:, 1])
        return np.exp(lo + u * (hi - lo))
    return b[:, 0] + u * (b[:, 1] - b[:, 0])


# ---------------------------------------------------------------- 3D assembly

def _node_axes(n):
    """(k, j, i) index grids over the (n+1)^3 nodes, x fastest on ravel."""
    idx = np.arange(n + 1)
    return np.meshgrid(idx, idx, idx, indexing="ij")


def _overlap(lo, hi, a, b):
    return np.maximum(0.0, np.minimum(hi, b) - np.maximum(lo, a))


def _face_weights(spec: FDProblemSpec, n: int, q: int, d: int) -> np.ndarray:
    """Edge weights of term q for edges X -> X + e_d, over all nodes with X_d < n.

    Returned as a full (n+1)^3 array (zero where X_d = n).
    """
    h = 1.0 / n
    K, J, I = _node_axes(n)
    coords = [I * h, J * h, K * h]          # x, y, z of each node
    mid = [c.astype(np.float64).copy() for c in coords]
    mid[d] = mid[d] + 0.5 * h               # edge midpoint
    valid = [I, J, K][d] < n
    if spec.kind == "thermal-block":
        bx, by, bz = spec.blocks
        nb = (bx, by, bz)
        a, rem = q % bx, q // bx
        b, c = rem % by, rem // by
        cell = (a, b, c)
        w = np.ones_like(mid[0])
        for ax in range(3):
            lo, hi = cell[ax] / nb[ax], (cell[ax] + 1) / nb[ax]
            if ax == d:
                w = w * ((mid[ax] >= lo) & (mid[ax] < hi))
            else:
                w = w * (_overlap(mid[ax] - 0.5 * h, mid[ax] + 0.5 * h, lo, hi) / h)
        w = h * w
    else:
        if q == 0:
            w = np.full(mid[0].shape, h)
        else:
            k = q
            w = h * (np.sin(k * np.pi * mid[0]) * np.sin(k * np.pi * mid[1])
                     * np.cos(k * np.pi * mid[2]))
    return np.where(valid, w, 0.0)


def assemble_term_full(spec: FDProblemSpec, n: int, q: int) -> sp.csr_matrix:
    """Term-q operator on all (n+1)^3 nodes (edge-Laplacian with weights)."""
    nn = (n + 1) ** 3
    strides = (1, n + 1, (n + 1) ** 2)
    rows, cols, vals = [], [], []
    K, J, I = _node_axes(n)
    ids = (I + (n + 1) * (J + (n + 1) * K)).ravel()
    for d in range(3):
        w = _face_weights(spec, n, q, d).ravel()
        mask = ([I, J, K][d] < n).ravel()
        a = ids[mask]
        b = a + strides[d]
        ww = w[mask]
        rows += [a, b, a, b]
        cols += [a, b, b, a]
        vals += [ww, ww, -ww, -ww]
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(nn, nn))
    return A.tocsr()


def interior_mask(n: int) -> np.ndarray:
    """Dirichlet mask on lexicographic nodes (reference problems.py:63-75)."""
    K, J, I = _node_axes(n)
    on_b = (I == 0) | (I == n) | (J == 0) | (J == n) | (K == 0) | (K == n)
    return on_b.ravel()


def rhs_full(spec: FDProblemSpec, n: int) -> np.ndarray:
    """Nodal load h^3 f(X) on all nodes."""
    h = 1.0 / n
    K, J, I = _node_axes(n)
    if spec.kind == "thermal-block":
        f = np.ones(I.shape)
    else:
        r2 = (I * h - 0.5) ** 2 + (J * h - 0.5) ** 2 + (K * h - 0.5) ** 2
        f = np.exp(-r2 / 0.02)
    return (h ** 3 * f).ravel()


def prolongation_full(nc: int) -> sp.csr_matrix:
    """Trilinear interpolation nc -> 2nc cells on all nodes (reference grid.py:131-141)."""
    nf = 2 * nc
    r = np.arange(nf + 1)
    # fine node r sits on coarse r/2 (even) or between (r-1)/2 and (r+1)/2 (odd)
    rows = np.concatenate([r[r % 2 == 0], r[r % 2 == 1], r[r % 2 == 1]])
    cols = np.concatenate([r[r % 2 == 0] // 2, (r[r % 2 == 1] - 1) // 2,
                           (r[r % 2 == 1] + 1) // 2])
    vals = np.concatenate([np.ones((nf + 2) // 2), np.full(nf // 2, 0.5),
                           np.full(nf // 2, 0.5)])
    P1 = sp.csr_matrix((vals, (rows, cols)), shape=(nf + 1, nc + 1))
    return sp.kron(sp.kron(P1, P1), P1).tocsr()


class OracleProblem:
    """Affine operator factory over a nested hierarchy (reference grid.py:193-290).

    Terms are assembled on the finest grid, restricted to free DoFs, and
    Galerkin-coarsened term by term; operator(mu, level) is the theta-weighted
    sum accumulated in term order, exactly as grid.py:246-255.
    """

    def __init__(self, spec: FDProblemSpec, n: int, m0: int = 4):
        if n % m0 or (n // m0) & (n // m0 - 1):
            raise ValueError("n must be m0 * 2^J")
        if spec.kind == "thermal-block" and any(n % b for b in spec.blocks):
            raise ValueError("block interfaces must fall on grid planes")
        self.spec = spec
        self.n = n
        self.m0 = m0
        cells = [m0]
        while cells[-1] < n:
            cells.append(cells[-1] * 2)
        if len(cells) < 2:
            raise ValueError("need at least 2 levels for coarse-grid correction")
        self.cells = tuple(cells)
        self.free_by_level = [np.flatnonzero(~interior_mask(c)) for c in self.cells]
        self.free = self.free_by_level[-1]
        self.n_free = len(self.free)
        self.terms_full = [assemble_term_full(spec, n, q) for q in range(spec.n_terms)]
        self.terms_ff = [T[self.free][:, self.free].tocsr() for T in self.terms_full]
        self.prolongations = []
        for i in range(len(self.cells) - 1):
            P = prolongation_full(self.cells[i])
            self.prolongations.append(
                P[self.free_by_level[i + 1]][:, self.free_by_level[i]].tocsr())
        from .solvers import galerkin
        self.terms_by_level = [None] * len(self.cells)
        self.terms_by_level[-1] = self.terms_ff
        for i in range(len(self.cells) - 2, -1, -1):
            P = self.prolongations[i]
            self.terms_by_level[i] = [galerkin(T, P) for T in self.terms_by_level[i + 1]]
        self._rhs = rhs_full(spec, n)[self.free]

    @property
    def levels(self) -> int:
        return len(self.cells)

    def operator(self, mu, level=None) -> sp.csr_matrix:
        if level is None:
            level = self.levels - 1
        th = self.spec.theta(mu)
        terms = self.terms_by_level[level]
        A = th[0] * terms[0]
        for t, T in zip(th[1:], terms[1:]):
            A = A + t * T
        return A.tocsr()

    def operator_rows(self, mu, rows) -> sp.csr_matrix:
        rows = list(rows)
        th = self.spec.theta(mu)
        out = th[0] * self.terms_ff[0][rows, :]
        for t, T in zip(th[1:], self.terms_ff[1:]):
            out = out + t * T[rows, :]
        return out.tocsr()

    def rhs(self, mu=None) -> np.ndarray:
        if mu is not None:
            self.spec.check_mu(mu)
        return self._rhs.copy()


def interior_to_padded(v: np.ndarray, n: int) -> np.ndarray:
    """Map an interior-ordered vector to the product's padded (pitch n) layout."""
    m = n - 1
    out = np.zeros((n, n, n))
    out[1:, 1:, 1:] = np.asarray(v).reshape(m, m, m)
    return out.ravel()


def padded_to_interior(v: np.ndarray, n: int) -> np.ndarray:
    return np.asarray(v).reshape(n, n, n)[1:, 1:, 1:].ravel().copy()
