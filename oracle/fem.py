"""Oracle for the reference's assembled Q1 FEM problems — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's trilinear hexahedral assembly and affine
problem factory, element by element in sparse (COO) form as the reference
does it, so it is independent of the product's stencil-direct assembly
(paper_2311_13862_b200/fem.py):

* 2x2x2 Gauss rule on [0,1]^3, trilinear shape values / gradients at the 8
  points (reference grid.py:17-58);
* element stiffness of one term: sum over points of w_g h^3 kappa(x_g)
  grad(phi_a) . diag(aniso) grad(phi_b) (grid.py:92-113), load with the same
  rule (grid.py:116-128);
* free DoFs = nodes off the Dirichlet boundary (problems.py:63-75), free-DoF
  trilinear prolongations (grid.py:131-141), termwise Galerkin coarsening
  P^T (A P) (grid.py:173-182, 222-236), operator(mu, level) = sum_q theta_q A_q in
  term order (grid.py:246-255), rhs = load - sum_q theta_q A_q[free, dir] g
  (grid.py:266-284).

Pinned against tests/golden/golden_fem.npz (the unmodified reference run on
``example-1``, tests/golden/make_golden.py --fem) and golden_fem2.npz
(``example-2``: zero-flux face, anisotropy, plane smoothers; ``--fem2``).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

_PTS = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])


def _corners():
    return [(l & 1, (l >> 1) & 1, (l >> 2) & 1) for l in range(8)]


def shape_tables():
    """vals[g, l], grads[g, axis, l] (reference coordinates) and weights w[g]."""
    vals = np.zeros((8, 8))
    grads = np.zeros((8, 3, 8))
    w = np.full(8, 0.125)
    for g, (gx, gy, gz) in enumerate(_corners()):
        t = (_PTS[gx], _PTS[gy], _PTS[gz])
        for l, c in enumerate(_corners()):
            ph = [t[a] if c[a] else 1.0 - t[a] for a in range(3)]
            dph = [1.0 if c[a] else -1.0 for a in range(3)]
            vals[g, l] = ph[0] * ph[1] * ph[2]
            grads[g, 0, l] = dph[0] * ph[1] * ph[2]
            grads[g, 1, l] = ph[0] * dph[1] * ph[2]
            grads[g, 2, l] = ph[0] * ph[1] * dph[2]
    return vals, grads, w


def _elements(n):
    e = np.arange(n)
    ez, ey, ex = np.meshgrid(e, e, e, indexing="ij")
    return ex.ravel(), ey.ravel(), ez.ravel()


def element_nodes(n):
    ex, ey, ez = _elements(n)
    return np.stack([(ex + cx) + (n + 1) * ((ey + cy) + (n + 1) * (ez + cz))
                     for cx, cy, cz in _corners()], axis=1)


def gauss_points(n):
    h = 1.0 / n
    ex, ey, ez = _elements(n)
    c = np.array(_corners())
    return ((ex[:, None] + _PTS[c[:, 0]][None]) * h, (ey[:, None] + _PTS[c[:, 1]][None]) * h,
            (ez[:, None] + _PTS[c[:, 2]][None]) * h)


def stiffness(n, kernel, aniso=(1.0, 1.0, 1.0)) -> sp.csr_matrix:
    h = 1.0 / n
    _, grads, w = shape_tables()
    Kg = np.zeros((8, 8, 8))
    for g in range(8):
        G = grads[g] / h
        Kg[g] = w[g] * h ** 3 * sum(aniso[a] * np.outer(G[a], G[a]) for a in range(3))
    kv = kernel(*gauss_points(n))
    kv = np.broadcast_to(np.asarray(kv, dtype=np.float64), (n ** 3, 8))
    elem = np.tensordot(kv, Kg, axes=([1], [0]))        # (e, 8, 8)
    conn = element_nodes(n)
    nn = (n + 1) ** 3
    rows = np.repeat(conn, 8, axis=1).ravel()
    cols = np.tile(conn, (1, 8)).ravel()
    return sp.coo_matrix((elem.ravel(), (rows, cols)), shape=(nn, nn)).tocsr()


def load(n, source, mu) -> np.ndarray:
    h = 1.0 / n
    vals, _, w = shape_tables()
    fv = source(*gauss_points(n), mu)
    fv = np.broadcast_to(np.asarray(fv, dtype=np.float64), (n ** 3, 8))
    elem = fv @ (w[:, None] * h ** 3 * vals)
    out = np.zeros((n + 1) ** 3)
    np.add.at(out, element_nodes(n).ravel(), elem.ravel())
    return out


def dirichlet_nodes(n, neumann_face_x1=False) -> np.ndarray:
    i = np.arange(n + 1)
    kz, ky, kx = np.meshgrid(i, i, i, indexing="ij")
    b = (kx == 0) | (kx == n) | (ky == 0) | (ky == n) | (kz == 0) | (kz == n)
    if neumann_face_x1:
        b &= kx != n
    return b.ravel()


def prolongation(nc) -> sp.csr_matrix:
    nf = 2 * nc
    r = list(range(0, nf + 1, 2)) + list(range(1, nf, 2)) * 2
    c = list(range(nc + 1)) + list(range(nc)) + list(range(1, nc + 1))
    v = [1.0] * (nc + 1) + [0.5] * (2 * nc)
    P1 = sp.csr_matrix((v, (r, c)), shape=(nf + 1, nc + 1))
    return sp.kron(sp.kron(P1, P1), P1).tocsr()


# ------------------------------------------------------------------ example-1 (problems.py:78-113)

class Example1:
    pid = "example-1"
    p = 2
    bounds = np.array([[0.0, 2.0], [0.0, 1.0]])
    neumann_face_x1 = False
    aniso = ((1.0, 1.0, 1.0), (1.0, 1.0, 1.0))

    @staticmethod
    def _rad(x, y, z):
        return 4.0 * (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2

    def kernels(self):
        return (lambda x, y, z: np.ones(np.shape(x)),
                lambda x, y, z: np.sin(20.0 * np.pi * self._rad(x, y, z)) ** 2)

    def theta(self, mu):
        return np.array([1.0, mu[0]])

    def source(self, x, y, z, mu):
        return 3.0 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)

    def dirichlet(self, x, y, z, mu):
        return ((1.0 - mu[1]) * np.cos(10.0 * np.pi * self._rad(x, y, z))
                + mu[1] * np.cos(10.0 * np.pi * (x + y + z)))

    def check_mu(self, mu):
        mu = np.asarray(mu, dtype=np.float64)
        if mu.shape != (self.p,) or np.any(mu < self.bounds[:, 0]) or np.any(mu > self.bounds[:, 1]):
            raise ValueError("parameter outside bounds")
        return mu


# ------------------------------------------------------------------ example-2 (problems.py:113-152)

def _indicator(y_lo, y_hi, z_lo, z_hi):
    """Block indicator of the y/z quadrant (problems.py:116-122)."""
    def kernel(x, y, z):
        return (((y >= y_lo) & (y < y_hi)) & ((z >= z_lo) & (z < z_hi))).astype(np.float64)
    return kernel


class Example2:
    """Mixed problem: zero-flux face x = 1, anisotropic diag(1, 1, 1e-2) piecewise-constant
    coefficient on four y/z quadrants, mu-dependent Gaussian source (problems.py:135-152)."""

    pid = "example-2"
    p = 7
    bounds = np.array([[0.1, 1.0]] * 3 + [[0.4, 0.6]] * 3 + [[0.25, 0.5]])
    neumann_face_x1 = True
    aniso = ((1.0, 1.0, 1.0e-2),) * 4

    def kernels(self):
        return (_indicator(0.0, 0.5, 0.0, 0.5), _indicator(0.0, 0.5, 0.5, 1.01),
                _indicator(0.5, 1.01, 0.0, 0.5), _indicator(0.5, 1.01, 0.5, 1.01))

    def theta(self, mu):
        return np.array([mu[0], mu[1], mu[2], 1.0])

    def source(self, x, y, z, mu):
        r2 = (x - mu[3]) ** 2 + (y - mu[4]) ** 2 + (z - mu[5]) ** 2
        return mu[6] + np.exp(-r2 / mu[6]) / mu[6]

    def dirichlet(self, x, y, z, mu):
        return np.zeros(np.broadcast(x, y, z).shape)

    check_mu = Example1.check_mu


class OracleFemProblem:
    """Reference ParametricProblem restated for assembled problems (grid.py:193-290)."""

    def __init__(self, spec, levels=3, m0=2):
        self.spec = spec
        self.cells = tuple(m0 * 2 ** i for i in range(levels))
        self.n = n = self.cells[-1]
        self.free_by_level, self.dir_by_level = [], []
        for c in self.cells:
            d = dirichlet_nodes(c, spec.neumann_face_x1)
            self.free_by_level.append(np.flatnonzero(~d))
            self.dir_by_level.append(np.flatnonzero(d))
        free, dirn = self.free_by_level[-1], self.dir_by_level[-1]
        full = [stiffness(n, k, a) for k, a in zip(spec.kernels(), spec.aniso)]
        self.terms_fd = [T[free][:, dirn].tocsr() for T in full]
        self.prolongations = [prolongation(self.cells[i])[self.free_by_level[i + 1]]
                              [:, self.free_by_level[i]].tocsr() for i in range(levels - 1)]
        self.terms_by_level = [None] * levels
        self.terms_by_level[-1] = [T[free][:, free].tocsr() for T in full]
        for i in range(levels - 2, -1, -1):
            P = self.prolongations[i]
            self.terms_by_level[i] = [(P.T @ (T @ P)).tocsr() for T in self.terms_by_level[i + 1]]
        self.terms_ff = self.terms_by_level[-1]
        # example-1's source is mu-independent (assembled once, grid.py:270-275)
        self._load = None if spec.neumann_face_x1 else load(n, spec.source, None)
        # z-layer of every free DoF per level (plane smoothers, multigrid.py:197-201)
        self.layers_by_level = [f // (c + 1) ** 2 for f, c in zip(self.free_by_level, self.cells)]

    @property
    def levels(self):
        return len(self.cells)

    def operator(self, mu, level=None):
        if level is None:
            level = self.levels - 1
        th = self.spec.theta(self.spec.check_mu(mu))
        T = self.terms_by_level[level]
        A = th[0] * T[0]
        for t, M in zip(th[1:], T[1:]):
            A = A + t * M
        return A.tocsr()

    def operator_rows(self, mu, rows):
        rows = list(rows)
        th = self.spec.theta(self.spec.check_mu(mu))
        out = th[0] * self.terms_ff[0][rows, :]
        for t, T in zip(th[1:], self.terms_ff[1:]):
            out = out + t * T[rows, :]
        return out.tocsr()

    def rhs(self, mu):
        mu = self.spec.check_mu(mu)
        n = self.n
        ld = self._load if self._load is not None else load(n, self.spec.source, mu)
        f = ld[self.free_by_level[-1]].copy()
        t = np.linspace(0.0, 1.0, n + 1)
        Z, Y, X = np.meshgrid(t, t, t, indexing="ij")
        d = self.dir_by_level[-1]
        g = self.spec.dirichlet(X.ravel()[d], Y.ravel()[d], Z.ravel()[d], mu)
        for th, T in zip(self.spec.theta(mu), self.terms_fd):
            f -= th * (T @ g)
        return f
