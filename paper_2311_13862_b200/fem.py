"""Assembled (trilinear FEM) problems of the reference on the B200 path.

The reference's own test problems (problems.py:78-155: ``example-1``,
``example-2``) are hexahedral Q1 finite-element discretisations: per affine
term a stiffness matrix assembled once on the finest grid with a 2x2x2 Gauss
rule (grid.py:92-113), restricted to the free DoFs and Galerkin-coarsened
term by term (grid.py:203-236); ``operator(mu, level) = sum_q theta_q A_q``
(grid.py:246-255) and ``rhs(mu)`` = load minus the lifted Dirichlet data
(grid.py:266-284).

Here the mu-independent part is built once on the host and handed to the
native library as per-term symmetric 27-point coefficient arrays on every
level (``rbws_hierarchy_create_stored``); per-parameter operators exist only
on the device, batched (``stored_combine``).  Assembly is stencil-direct: the
element matrix of every (node, offset) pair is accumulated straight into the
27 coefficient planes of the node, never into a sparse matrix; only the
Galerkin triple products go through scipy.

Scope: Dirichlet problems (free DoFs = interior nodes, the padded layout of
the separable path).  ``example-2``'s zero-flux face keeps boundary nodes free
and its default smoother is the plane-block Jacobi of multigrid.py:48-110: it
runs on the full-node path (``fem_fn.py``), to which ``ParametricProblem``
dispatches; ``FemProblem`` itself refuses it (NotImplementedError).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import scipy.sparse as sp

from . import _native
from .grid import padded_len

# ------------------------------------------------------------------ problem definitions


@dataclass(frozen=True)
class DiffusionTerm:
    """One affine component theta(mu) * kernel(x) * diag(aniso) of the diffusion tensor."""

    theta: Callable
    kernel: Callable
    aniso: tuple = (1.0, 1.0, 1.0)


@dataclass(frozen=True)
class FemProblemSpec:
    """A parametrised diffusion BVP on (0,1)^3 (reference ProblemSpec, problems.py:26-75)."""

    pid: str
    p: int
    bounds: np.ndarray
    diffusion_terms: Sequence[DiffusionTerm]
    source: Callable
    dirichlet: Callable
    neumann_face_x1: bool = False
    source_mu_dependent: bool = True
    kind: str = "fem"

    def __post_init__(self):
        b = np.asarray(self.bounds, dtype=np.float64)
        if b.shape != (self.p, 2):
            raise ValueError("bounds must be (p, 2)")
        if np.any(b[:, 0] >= b[:, 1]):
            raise ValueError("each parameter range needs min < max")
        object.__setattr__(self, "bounds", b)

    @property
    def n_terms(self) -> int:
        return len(self.diffusion_terms)

    def check_mu(self, mu) -> np.ndarray:
        mu = np.asarray(mu, dtype=np.float64)
        if mu.shape != (self.p,):
            raise ValueError(f"{self.pid} expects {self.p}-dimensional parameters")
        if np.any(mu < self.bounds[:, 0]) or np.any(mu > self.bounds[:, 1]):
            raise ValueError(f"parameter {mu} outside {self.pid} bounds")
        return mu

    def check_mus(self, mus) -> np.ndarray:
        mus = np.atleast_2d(np.asarray(mus, dtype=np.float64))
        if mus.shape[1] != self.p:
            raise ValueError(f"{self.pid} expects {self.p}-dimensional parameters")
        if np.any(mus < self.bounds[:, 0]) or np.any(mus > self.bounds[:, 1]):
            raise ValueError(f"parameters outside {self.pid} bounds")
        return mus

    def thetas(self, mus) -> np.ndarray:
        mus = self.check_mus(mus)
        return np.array([[float(t.theta(m)) for t in self.diffusion_terms] for m in mus])


def _r2(x, y, z):
    return 4.0 * (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2


def example1() -> FemProblemSpec:
    """Dirichlet problem, isotropic oscillatory coefficient, p = 2 (problems.py:78-113)."""
    def one(x, y, z):
        return np.ones(np.broadcast(x, y, z).shape)

    def osc(x, y, z):
        return np.sin(20.0 * np.pi * _r2(x, y, z)) ** 2

    def source(x, y, z, mu):
        return 3.0 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)

    def dirichlet(x, y, z, mu):
        return ((1.0 - mu[1]) * np.cos(10.0 * np.pi * _r2(x, y, z))
                + mu[1] * np.cos(10.0 * np.pi * (x + y + z)))

    return FemProblemSpec(
        pid="example-1", p=2, bounds=np.array([[0.0, 2.0], [0.0, 1.0]]),
        diffusion_terms=(DiffusionTerm(lambda mu: 1.0, one),
                         DiffusionTerm(lambda mu: mu[0], osc)),
        source=source, dirichlet=dirichlet, neumann_face_x1=False,
        source_mu_dependent=False)


def example2() -> FemProblemSpec:
    """Mixed problem, piecewise-constant anisotropic coefficient, p = 7 (problems.py:116-155)."""
    an = (1.0, 1.0, 1.0e-2)

    def ind(y0, y1, z0, z1):
        def k(x, y, z):
            return (((y >= y0) & (y < y1)) & ((z >= z0) & (z < z1))).astype(np.float64)
        return k

    def source(x, y, z, mu):
        r2 = (x - mu[3]) ** 2 + (y - mu[4]) ** 2 + (z - mu[5]) ** 2
        return mu[6] + np.exp(-r2 / mu[6]) / mu[6]

    def dirichlet(x, y, z, mu):
        return np.zeros(np.broadcast(x, y, z).shape)

    return FemProblemSpec(
        pid="example-2", p=7,
        bounds=np.array([[0.1, 1.0]] * 3 + [[0.4, 0.6]] * 3 + [[0.25, 0.5]]),
        diffusion_terms=(DiffusionTerm(lambda mu: mu[0], ind(0.0, 0.5, 0.0, 0.5), an),
                         DiffusionTerm(lambda mu: mu[1], ind(0.0, 0.5, 0.5, 1.01), an),
                         DiffusionTerm(lambda mu: mu[2], ind(0.5, 1.01, 0.0, 0.5), an),
                         DiffusionTerm(lambda mu: 1.0, ind(0.5, 1.01, 0.5, 1.01), an)),
        source=source, dirichlet=dirichlet, neumann_face_x1=True, source_mu_dependent=True)


# ------------------------------------------------------------------ Q1 element data

_GP = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])  # 2-point Gauss on [0,1]


def _gauss_tables():
    """1D shape values v[g, a] = phi_a(t_g), derivatives d[a] (d/dt phi_a), local node
    triples (ax, ay, az) of the 8 element nodes (l = ax + 2 ay + 4 az) and Gauss triples
    (gx, gy, gz) of the 8 points (x fastest, grid.py:22-58's ordering)."""
    v = np.stack([1.0 - _GP, _GP], axis=1)      # [g][a]
    d = np.array([-1.0, 1.0])
    loc = np.array([(l & 1, (l >> 1) & 1, (l >> 2) & 1) for l in range(8)])
    return v, d, loc, loc.copy()


def _elem_stiffness_per_point(h: float, aniso) -> np.ndarray:
    """Kg[g, a, b]: the 8x8 element stiffness contribution of Gauss point g with unit
    coefficient: w_g h^3 sum_d aniso_d (dphi_a/dx_d)(dphi_b/dx_d), built from 1D tensor
    factors (gradient of phi_a along d = d[a_d]/h times the other two 1D values)."""
    v, d, loc, gp = _gauss_tables()
    K = np.zeros((8, 8, 8))
    w = 0.125 * h ** 3
    for g in range(8):
        gx = gp[g]
        grads = np.empty((8, 3))
        for a in range(8):
            vals = [v[gx[ax], loc[a][ax]] for ax in range(3)]
            for dd in range(3):
                gvals = list(vals)
                gvals[dd] = d[loc[a][dd]] / h
                grads[a, dd] = gvals[0] * gvals[1] * gvals[2]
        K[g] = w * (grads * np.asarray(aniso)[None, :]) @ grads.T
    return K


def _quad_points(n: int):
    """Physical Gauss-point coordinates of every element, shape (n^3, 8) per axis
    (elements x fastest, points in _gauss_tables order)."""
    h = 1.0 / n
    _, _, _, gp = _gauss_tables()
    e = np.arange(n)
    ez, ey, ex = np.meshgrid(e, e, e, indexing="ij")
    ex, ey, ez = ex.ravel(), ey.ravel(), ez.ravel()
    return ((ex[:, None] + _GP[gp[None, :, 0]]) * h, (ey[:, None] + _GP[gp[None, :, 1]]) * h,
            (ez[:, None] + _GP[gp[None, :, 2]]) * h)


def _o27(dx, dy, dz):
    return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)


def assemble_stencil(n: int, kernel, aniso=(1.0, 1.0, 1.0)) -> np.ndarray:
    """Full-node 27-point stiffness stencil of one term: S[o27, kz, ky, kx] on the
    (n+1)^3 nodes, S[o](X) = A[X, X + o] (stencil-direct Q1 assembly)."""
    h = 1.0 / n
    Kg = _elem_stiffness_per_point(h, aniso)
    xq, yq, zq = _quad_points(n)
    kv = kernel(xq, yq, zq)
    if np.isscalar(kv):
        kv = np.full(xq.shape, float(kv))
    kv = np.asarray(kv, dtype=np.float64).reshape(n, n, n, 8)   # [ez, ey, ex, g]
    _, _, loc, _ = _gauss_tables()
    S = np.zeros((27, n + 1, n + 1, n + 1))
    for a in range(8):
        ax, ay, az = loc[a]
        for b in range(8):
            bx, by, bz = loc[b]
            ke = kv @ Kg[:, a, b]                                   # [ez, ey, ex]
            S[_o27(bx - ax, by - ay, bz - az), az:az + n, ay:ay + n, ax:ax + n] += ke
    return S


def assemble_load_grid(n: int, source, mu) -> np.ndarray:
    """Load vector on the (n+1)^3 nodes as [kz, ky, kx] (2x2x2 Gauss rule)."""
    h = 1.0 / n
    v, _, loc, gp = _gauss_tables()
    xq, yq, zq = _quad_points(n)
    fv = source(xq, yq, zq, mu)
    if np.isscalar(fv):
        fv = np.full(xq.shape, float(fv))
    fv = np.asarray(fv, dtype=np.float64).reshape(n, n, n, 8)
    w = 0.125 * h ** 3
    out = np.zeros((n + 1, n + 1, n + 1))
    for a in range(8):
        ax, ay, az = loc[a]
        phi = np.array([v[gp[g][0], ax] * v[gp[g][1], ay] * v[gp[g][2], az] for g in range(8)])
        out[az:az + n, ay:ay + n, ax:ax + n] += fv @ (w * phi)
    return out


# ------------------------------------------------------------------ stencil <-> CSR

_FWD = [(dx, dy, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)] + [(-1, 1, 0), (0, 1, 0),
                                                                   (1, 1, 0), (1, 0, 0)]


def interior_csr(S: np.ndarray) -> sp.csr_matrix:
    """Free-free block (interior nodes, reference free-DoF order) of a full-node stencil."""
    n = S.shape[1] - 1
    m = n - 1
    idx = np.arange(m ** 3).reshape(m, m, m)
    rows, cols, vals = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                z0, z1 = max(0, -dz), m - max(0, dz)
                y0, y1 = max(0, -dy), m - max(0, dy)
                x0, x1 = max(0, -dx), m - max(0, dx)
                r = idx[z0:z1, y0:y1, x0:x1]
                c = idx[z0 + dz:z1 + dz, y0 + dy:y1 + dy, x0 + dx:x1 + dx]
                v = S[_o27(dx, dy, dz), 1 + z0:1 + z1, 1 + y0:1 + y1, 1 + x0:1 + x1]
                rows.append(r.ravel()); cols.append(c.ravel()); vals.append(v.ravel())
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(m ** 3, m ** 3))
    A.eliminate_zeros()
    return A


def csr_to_coef(A: sp.csr_matrix, n: int) -> np.ndarray:
    """Interior CSR on an n-cell grid -> [14][n^3] padded symmetric coefficients (the
    diagonal and the forward offsets of include/rbws_b200.h; zero on ghosts)."""
    m = n - 1
    C = sp.coo_matrix(A)
    r, c, v = C.row, C.col, C.data
    ri, rj, rk = r % m, (r // m) % m, r // (m * m)
    ci, cj, ck = c % m, (c // m) % m, c // (m * m)
    dx, dy, dz = ci - ri, cj - rj, ck - rk
    if np.any(np.abs(dx) > 1) or np.any(np.abs(dy) > 1) or np.any(np.abs(dz) > 1):
        raise ValueError("operator is not a 27-point stencil")
    out = np.zeros((14, n ** 3))
    X = (ri + 1) + n * ((rj + 1) + n * (rk + 1))
    diag = (dx == 0) & (dy == 0) & (dz == 0)
    out[0, X[diag]] = v[diag]
    for o, (ox, oy, oz) in enumerate(_FWD, start=1):
        sel = (dx == ox) & (dy == oy) & (dz == oz)
        out[o, X[sel]] = v[sel]
    return out


def _prolongation_free(nc: int) -> sp.csr_matrix:
    """Trilinear interpolation nc -> 2nc cells restricted to interior nodes."""
    nf = 2 * nc
    rows, cols, vals = [], [], []
    for i in range(1, nc):           # coarse interior 1..nc-1 -> fine interior 1..nf-1
        for fi, w in ((2 * i - 1, 0.5), (2 * i, 1.0), (2 * i + 1, 0.5)):
            rows.append(fi - 1); cols.append(i - 1); vals.append(w)
    P1 = sp.csr_matrix((vals, (rows, cols)), shape=(nf - 1, nc - 1))
    return sp.kron(sp.kron(P1, P1), P1).tocsr()


# ------------------------------------------------------------------ the problem factory


def rhs_from_stencils(spec: FemProblemSpec, stencils, n: int, mus, load=None) -> np.ndarray:
    """f_h(mu) (count, (n-1)^3): interior load minus the lifted Dirichlet data, term by term
    in term order (grid.py:266-284); the lifting sum_o S_q[o](X) g(X + o) runs over the
    full-node stencils (g is zero on free nodes).  `load`: cached mu-independent load."""
    mus = spec.check_mus(mus)
    t = np.linspace(0.0, 1.0, n + 1)
    Z, Y, X = np.meshgrid(t, t, t, indexing="ij")
    bnd = np.ones((n + 1,) * 3, dtype=bool)
    bnd[1:n, 1:n, 1:n] = False
    th = spec.thetas(mus)
    out = np.empty((len(mus), (n - 1) ** 3))
    for m, mu in enumerate(mus):
        ld = load if load is not None else assemble_load_grid(n, spec.source, mu)
        f = ld[1:n, 1:n, 1:n].copy()
        g = np.zeros((n + 1,) * 3)
        g[bnd] = spec.dirichlet(X[bnd], Y[bnd], Z[bnd], mu)
        for q, S in enumerate(stencils):
            lift = np.zeros((n - 1,) * 3)
            for dz in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        lift += (S[_o27(dx, dy, dz), 1:n, 1:n, 1:n]
                                 * g[1 + dz:n + dz, 1 + dy:n + dy, 1 + dx:n + dx])
            f -= th[m, q] * lift
        out[m] = f.ravel()
    return out


def host_hierarchy(spec: FemProblemSpec, cells):
    """mu-independent host part: per-term full-node stencils of the finest grid, their
    free-free blocks and the termwise Galerkin hierarchy P^T (A P) (grid.py:173-182,
    222-236).  Returns (stencils, terms_by_level, prolongations)."""
    n = cells[-1]
    stencils = [assemble_stencil(n, t.kernel, t.aniso) for t in spec.diffusion_terms]
    prolongations = [_prolongation_free(c) for c in cells[:-1]]
    terms = [None] * len(cells)
    terms[-1] = [interior_csr(S) for S in stencils]
    for i in range(len(cells) - 2, -1, -1):
        P = prolongations[i]
        terms[i] = [(P.T @ (T @ P)).tocsr() for T in terms[i + 1]]
    return stencils, terms, prolongations


class FemProblem:
    """Batched counterpart of the reference ParametricProblem for assembled problems
    (grid.py:193-290): same constructor, per-term assembly + termwise Galerkin coarsening
    once, operators and right-hand sides per parameter batch on the device."""

    stored = True  # stored-coefficient hierarchy: mu-dependent rhs, term products by apply

    def apply_bytes_per_node(self, ctx) -> float:
        """Algorithmic bytes per interior node and instance of one finest-level batched
        apply: x + y, plus one pass over the batch-shared term coefficients (14 Q doubles
        per node) spread over the batch — or 14 per-instance coefficients when the batch
        keeps its own copies (Q > 4 or RBWS_FEM_SHARED=0)."""
        import os
        q = self.spec.n_terms
        shared = q <= 4 and os.environ.get("RBWS_FEM_SHARED", "1") != "0"
        return 16.0 + (112.0 * q / ctx.count if shared else 112.0)

    def __init__(self, spec: FemProblemSpec, levels: int = 3, m0: int = 2):
        if levels < 2:
            raise ValueError("need at least 2 levels for coarse-grid correction")
        if m0 < 2:
            raise ValueError("base grid needs at least 2 cells per dimension")
        if spec.neumann_face_x1:
            raise NotImplementedError(
                f"{spec.pid}: zero-flux faces (free boundary nodes) are not on the B200 path")
        _native.require_cuda()
        self.spec = spec
        self.m0 = m0
        self.cells = tuple(m0 * 2 ** i for i in range(levels))
        self.n = n = self.cells[-1]
        self.n_free = (n - 1) ** 3
        self._stencils, self.terms_by_level, self.prolongations = host_hierarchy(
            spec, self.cells)
        coef = np.concatenate([csr_to_coef(T, self.cells[l]).ravel()
                               for l in range(levels) for T in self.terms_by_level[l]])
        h = ctypes.c_void_p()
        _native.call("rbws_hierarchy_create_stored", ctypes.byref(h), n, m0, spec.n_terms,
                     coef.ctypes.data)
        self._h = h
        self._load = None
        self._dirichlet_nodes = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _native._lib is not None:
            _native._lib.rbws_hierarchy_destroy(h)

    @property
    def handle(self):
        return self._h

    @property
    def levels(self) -> int:
        return len(self.cells)

    @property
    def finest_level(self) -> int:
        return self.levels - 1

    @property
    def finest_cells(self) -> int:
        return self.n

    def thetas(self, mus):
        import torch
        return torch.as_tensor(self.spec.thetas(mus), dtype=torch.float64, device="cuda")

    def operator_host(self, mu, level: int | None = None) -> sp.csr_matrix:
        """A_h(mu) on the free DoFs of `level` as a host CSR (grid.py:246-255)."""
        if level is None:
            level = self.finest_level
        th = self.spec.thetas([mu])[0]
        T = self.terms_by_level[level]
        A = th[0] * T[0]
        for t, M in zip(th[1:], T[1:]):
            A = A + t * M
        return A.tocsr()

    def rhs_host(self, mus) -> np.ndarray:
        """f_h(mu) (count, (n-1)^3) in the reference's free-DoF order."""
        if self._load is None and not self.spec.source_mu_dependent:
            self._load = assemble_load_grid(self.n, self.spec.source, None)
        return rhs_from_stencils(self.spec, self._stencils, self.n, mus, self._load)

    def rhs(self, mus):
        """Padded batch of f_h(mu) on the device (one instance per parameter)."""
        from .grid import to_padded
        return to_padded(self.rhs_host(mus), self.n)

    def zeros(self, count: int, level: int | None = None):
        import torch
        n = self.cells[self.finest_level if level is None else level]
        return torch.zeros(padded_len(n, count), dtype=torch.float64, device="cuda")

    def operator(self, mus, ctx=None):
        from .grid import BatchOperator
        from .multigrid import mg_context_for
        if ctx is None:
            ctx = mg_context_for(self, mus)
        return BatchOperator(ctx)

    def term_apply(self, term: int, x, count: int, level: int | None = None):
        """y = A_term x for `count` padded vectors (mu-independent term product)."""
        import torch
        lvl = self.finest_level if level is None else level
        y = torch.zeros_like(x)
        _native.call("rbws_hierarchy_term_apply", self._h, lvl, term, count, x.data_ptr(),
                     y.data_ptr(), _native.stream_ptr())
        return y
