"""Assembled problems with free boundary nodes on the B200 path (full-node layout).

The reference's ``example-2`` (problems.py:135-152) keeps its zero-flux face x = 1
free, edge nodes included (problems.py:63-75), so its free DoFs do not fit the
padded interior layout of the separable / example-1 path.  Here every level stores
all (c+1)^3 nodes per instance with Dirichlet nodes held at zero
(``csrc/planes.cu``):

* host, once: per-term full-node Q1 stencils (``fem.assemble_stencil``), their
  free-free blocks, termwise Galerkin coarsening with the free-DoF trilinear
  prolongations (grid.py:131-141, 203-236), each level's terms as full-node 27-point
  coefficient arrays;
* device, per parameter batch (``mg_context_for``, multigrid.py:191-202):
  theta-combined coefficients per level, the z-plane blocks of every level >= 1
  (plane smoothers, multigrid.py:48-110) and the whole coarsest level as banded
  SPD systems, factored by banded Cholesky;
* ``mg_vcycle`` (multigrid.py:205-222) and the batched PCG ``mgcg_solve``
  (krylov.py:42-109) over those kernels.  Smoothers: ``"plane-jacobi"`` (the
  reference default for anisotropic terms, omega 0.6), ``"plane-z"`` (block
  Gauss-Seidel over the planes, ascending before / descending after the coarse
  correction; a parity path: 2 launches per plane) and ``"jacobi"`` (omega 0.7).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import scipy.sparse as sp

from . import _native
from .fem import FemProblemSpec, _o27, assemble_load_grid, assemble_stencil
from .krylov import OperatorError, SolveReports

JACOBI_OMEGA = 0.7   # multigrid.py:27
PLANE_OMEGA = 0.6    # multigrid.py:29


def free_mask(c: int, neumann_face_x1: bool) -> np.ndarray:
    """Free nodes of a c-cell level as a [kz][ky][kx] bool grid (problems.py:63-75)."""
    i = np.arange(c + 1)
    kz, ky, kx = np.meshgrid(i, i, i, indexing="ij")
    bnd = (kx == 0) | (kx == c) | (ky == 0) | (ky == c) | (kz == 0) | (kz == c)
    if neumann_face_x1:
        bnd &= kx != c
    return ~bnd


def full_csr(S: np.ndarray) -> sp.csr_matrix:
    """Full-node CSR of a [27][c+1][c+1][c+1] stencil (S[o](X) = A[X, X+o])."""
    c1 = S.shape[1]
    idx = np.arange(c1 ** 3).reshape(c1, c1, c1)
    rows, cols, vals = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                z0, z1 = max(0, -dz), c1 - max(0, dz)
                y0, y1 = max(0, -dy), c1 - max(0, dy)
                x0, x1 = max(0, -dx), c1 - max(0, dx)
                rows.append(idx[z0:z1, y0:y1, x0:x1].ravel())
                cols.append(idx[z0 + dz:z1 + dz, y0 + dy:y1 + dy, x0 + dx:x1 + dx].ravel())
                vals.append(S[_o27(dx, dy, dz), z0:z1, y0:y1, x0:x1].ravel())
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(c1 ** 3,) * 2)
    A.eliminate_zeros()
    return A


def fn_coef(A: sp.csr_matrix, free: np.ndarray, c: int) -> np.ndarray:
    """Free-DoF CSR of a c-cell level -> full-node coefficients [27][(c+1)^3]."""
    c1 = c + 1
    C = sp.coo_matrix(A)
    r, q = free[C.row], free[C.col]
    rx, ry, rz = r % c1, (r // c1) % c1, r // (c1 * c1)
    dx, dy, dz = q % c1 - rx, (q // c1) % c1 - ry, q // (c1 * c1) - rz
    if np.any(np.abs(dx) > 1) or np.any(np.abs(dy) > 1) or np.any(np.abs(dz) > 1):
        raise ValueError("operator is not a 27-point stencil")
    out = np.zeros((27, c1 ** 3))
    out[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1), r] = C.data
    return out


def prolongation_free(cc: int, free_c: np.ndarray, free_f: np.ndarray) -> sp.csr_matrix:
    """Trilinear cc -> 2cc prolongation on free DoFs (grid.py:131-141)."""
    nf = 2 * cc
    r = list(range(0, nf + 1, 2)) + list(range(1, nf, 2)) * 2
    col = list(range(cc + 1)) + list(range(cc)) + list(range(1, cc + 1))
    v = [1.0] * (cc + 1) + [0.5] * (2 * cc)
    P1 = sp.csr_matrix((v, (r, col)), shape=(nf + 1, cc + 1))
    return sp.kron(sp.kron(P1, P1), P1).tocsr()[free_f][:, free_c].tocsr()


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class FnFemProblem:
    """Batched counterpart of the reference ParametricProblem (grid.py:193-290) for
    assembled problems in the full-node layout (any Dirichlet mask)."""

    def __init__(self, spec: FemProblemSpec, levels: int = 3, m0: int = 2,
                 host_only: bool = False):
        """host_only: build the mu-independent host hierarchy only (no device arrays;
        for the host-side checks and the C-ABI-free tests)."""
        if levels < 2:
            raise ValueError("need at least 2 levels for coarse-grid correction")
        if m0 < 2:
            raise ValueError("base grid needs at least 2 cells per dimension")
        if not host_only:
            _native.require_cuda()
        self.spec = spec
        self.cells = tuple(m0 * 2 ** i for i in range(levels))
        self.n = n = self.cells[-1]
        self.masks = [free_mask(c, spec.neumann_face_x1).ravel() for c in self.cells]
        self.free_by_level = [np.flatnonzero(m) for m in self.masks]
        self.n_free = len(self.free_by_level[-1])
        self._stencils = [assemble_stencil(n, t.kernel, t.aniso) for t in spec.diffusion_terms]
        full = [full_csr(S) for S in self._stencils]
        free, dirn = self.free_by_level[-1], np.flatnonzero(~self.masks[-1])
        self._terms_fd = [T[free][:, dirn].tocsr() for T in full]
        self.prolongations = [prolongation_free(self.cells[i], self.free_by_level[i],
                                                self.free_by_level[i + 1])
                              for i in range(levels - 1)]
        terms = [None] * levels
        terms[-1] = [T[free][:, free].tocsr() for T in full]
        for i in range(levels - 2, -1, -1):
            P = self.prolongations[i]
            terms[i] = [(P.T @ (T @ P)).tocsr() for T in terms[i + 1]]
        self.terms_by_level = terms
        self._load = None
        if host_only:
            return
        import torch
        dev = "cuda"
        self._coef = [torch.as_tensor(np.stack([fn_coef(T, self.free_by_level[l], self.cells[l])
                                                for T in terms[l]]), device=dev)
                      for l in range(levels)]
        self._mask_dev = [torch.as_tensor(m.astype(np.uint8), device=dev) for m in self.masks]

    @property
    def levels(self) -> int:
        return len(self.cells)

    @property
    def handle(self):
        """No native hierarchy object: full-node problems run through FnMgContext (fem_fn),
        not the padded-layout batch entry points (rbws_batch_*)."""
        raise NotImplementedError(
            f"{self.spec.pid}: full-node problems have no padded-layout hierarchy handle; "
            "use mg_context_for / mgcg_solve / rbi_pcg_solve / l1roc_* (fem_fn contexts)")

    def thetas(self, mus):
        import torch
        return torch.as_tensor(self.spec.thetas(mus), dtype=torch.float64, device="cuda")

    def nodes(self, level=None) -> int:
        c = self.cells[-1 if level is None else level]
        return (c + 1) ** 3

    # ---------------------------------------------------------------- host views
    def operator_host(self, mu, level=None) -> sp.csr_matrix:
        level = self.levels - 1 if level is None else level
        th = self.spec.thetas([mu])[0]
        T = self.terms_by_level[level]
        A = th[0] * T[0]
        for t, M in zip(th[1:], T[1:]):
            A = A + t * M
        return A.tocsr()

    def rhs_host(self, mus) -> np.ndarray:
        """f_h(mu) (count, n_free): load minus lifted Dirichlet data (grid.py:266-284)."""
        mus = self.spec.check_mus(mus)
        n = self.n
        free, dirn = self.free_by_level[-1], np.flatnonzero(~self.masks[-1])
        t = np.linspace(0.0, 1.0, n + 1)
        Z, Y, X = (a.ravel() for a in np.meshgrid(t, t, t, indexing="ij"))
        th = self.spec.thetas(mus)
        out = np.empty((len(mus), len(free)))
        for m, mu in enumerate(mus):
            if self.spec.source_mu_dependent or self._load is None:
                ld = assemble_load_grid(n, self.spec.source, mu).ravel()
                if not self.spec.source_mu_dependent:
                    self._load = ld
            else:
                ld = self._load
            f = ld[free].copy()
            g = self.spec.dirichlet(X[dirn], Y[dirn], Z[dirn], mu)
            for q, T in enumerate(self._terms_fd):
                f -= th[m, q] * (T @ g)
            out[m] = f
        return out

    # ---------------------------------------------------------------- layout
    def to_full(self, v, level=None):
        """(count, n_free) free-DoF vectors -> (count, (c+1)^3) device tensor."""
        import torch
        level = self.levels - 1 if level is None else level
        v = torch.as_tensor(np.atleast_2d(np.asarray(v, dtype=np.float64)))
        out = torch.zeros(v.shape[0], self.nodes(level), dtype=torch.float64)
        out[:, torch.as_tensor(self.free_by_level[level])] = v
        return out.cuda()

    def from_full(self, t, level=None) -> np.ndarray:
        level = self.levels - 1 if level is None else level
        return t.detach().cpu().numpy()[:, self.free_by_level[level]]

    def rhs(self, mus):
        return self.to_full(self.rhs_host(mus))


class FnMgContext:
    """Batched MgContext (multigrid.py:116-129) of an FnFemProblem."""

    def __init__(self, problem: FnFemProblem, mus, nu: int = 1, smoother: str = "auto"):
        import torch
        if nu < 0:
            raise ValueError("smoothing count must be non-negative")
        if smoother == "auto":  # multigrid.py:183-188
            aniso = any(len(set(t.aniso)) > 1 for t in problem.spec.diffusion_terms)
            smoother = "plane-jacobi" if aniso else "jacobi"
        if smoother not in ("plane-jacobi", "plane-z", "jacobi"):
            raise ValueError(f"smoother {smoother!r} is not on the full-node B200 path")
        self.problem, self.nu, self.smoother = problem, nu, smoother
        self.omega = {"plane-jacobi": PLANE_OMEGA, "plane-z": 1.0}.get(smoother, JACOBI_OMEGA)
        mus = problem.spec.check_mus(mus)
        self.count = count = len(mus)
        self.mus = mus
        theta = torch.as_tensor(problem.spec.thetas(mus), dtype=torch.float64, device="cuda")
        Q = theta.shape[1]
        self.theta = theta
        import os
        # batch-shared finest apply: bitwise equal but measured slower at 64^3 x 64
        # (139.6 vs 158.2 solves/s, profiles/r01i_example2.md) -> opt-in RBWS_FN_SHARED=1
        self.shared_finest = Q <= 8 and os.environ.get("RBWS_FN_SHARED", "0") == "1"
        st = _native.stream_ptr()
        self.coefA, self.bands, self.bandsT = [], [], []
        # scatter-form plane solves on the transposed factors (rbws_fn_band_solve_t): opt-in,
        # RBWS_BAND_SOLVE_T=1 — measured slower than the gather-form kernel at 64^3 x 64
        # (MGCG 352-423 vs 287 ms, profiles/r02_example2.md)
        self.scatter = os.environ.get("RBWS_BAND_SOLVE_T", "0") == "1" and \
            smoother == "plane-jacobi"
        bad = []
        for l, c in enumerate(problem.cells):
            ca = torch.empty(count * 27 * problem.nodes(l), dtype=torch.float64, device="cuda")
            _native.call("rbws_fn_combine", count, Q, c, _ptr(theta), _ptr(problem._coef[l]),
                         _ptr(ca), st)
            self.coefA.append(ca)
            planar = 0 if l == 0 else (1 if smoother.startswith("plane") else -1)
            if planar < 0:
                self.bands.append(None)
                self.bandsT.append(None)
                continue
            nb = _native.load().rbws_fn_band_doubles(count, c, planar)
            band = torch.empty(nb, dtype=torch.float64, device="cuda")
            nsys = count * (c + 1) if planar else count
            info = torch.zeros(nsys, dtype=torch.int32, device="cuda")
            _native.call("rbws_fn_band_factor", count, c, planar, _ptr(ca), _ptr(band),
                         _ptr(info), st)
            self.bands.append(band)
            bandT = None
            if self.scatter and planar == 1:
                bandT = torch.empty_like(band)
                _native.call("rbws_fn_band_transpose", count, c, planar, _ptr(band),
                             _ptr(bandT), st)
            self.bandsT.append(bandT)
            bad.append((l, info))
        for l, info in bad:
            if int(info.max()) > 0:
                what = "coarsest operator" if l == 0 else "plane block"
                raise OperatorError(f"{what} not SPD (level {l})")

    @property
    def levels(self):
        return len(self.problem.cells)

    def apply(self, x, level=None, b=None, out=None):
        """A x (b None) or b - A x on `level` for the whole batch."""
        import torch
        level = self.levels - 1 if level is None else level
        y = torch.empty_like(x) if out is None else out
        bp = _ptr(b) if b is not None else None
        mode = 0 if b is None else 1
        if level == self.levels - 1 and self.shared_finest:
            # finest level: batch-shared term coefficients combined on the fly (bitwise the
            # per-instance apply; 16 B/node + the shared terms instead of 232 B/node)
            _native.call("rbws_fn_apply_shared", self.count, self.theta.shape[1],
                         self.problem.cells[level], _ptr(self.theta), _ptr(self.problem._coef[level]),
                         _ptr(x), bp, _ptr(y), mode, _native.stream_ptr())
        else:
            _native.call("rbws_fn_apply", self.count, self.problem.cells[level],
                         _ptr(self.coefA[level]), _ptr(x), bp, _ptr(y), mode, _native.stream_ptr())
        return y

    def _smooth(self, level, u, b, forward=True, from_zero=False):
        """nu sweeps on `level`; from_zero: u is the zero vector (the pre-smoothing of a V-cycle),
        so the first sweep's residual b - A u is b itself (bitwise) and no apply is launched."""
        c = self.problem.cells[level]
        st = _native.stream_ptr()
        if self.smoother == "plane-z":  # ascending pre / descending post (multigrid.py:97-110)
            import torch
            scratch = torch.empty(self.count * (c + 1) ** 2, dtype=torch.float64, device="cuda")
            for _ in range(self.nu):
                _native.call("rbws_fn_plane_gs_sweep", self.count, c, _ptr(self.coefA[level]),
                             _ptr(self.bands[level]), _ptr(b), _ptr(u), _ptr(scratch),
                             1 if forward else 0, st)
            return u
        for s in range(self.nu):
            r = b.clone() if (from_zero and s == 0) else self.apply(u, level, b)
            if self.smoother == "plane-jacobi":  # multigrid.py:91-95
                if self.bandsT[level] is not None:
                    _native.call("rbws_fn_band_solve_t", self.count, c, 1,
                                 _ptr(self.bands[level]), _ptr(self.bandsT[level]), _ptr(r),
                                 _ptr(u), self.omega, 1, st)
                else:
                    _native.call("rbws_fn_band_solve", self.count, c, 1, _ptr(self.bands[level]),
                                 _ptr(r), _ptr(u), self.omega, 1, st)
            else:
                _native.call("rbws_fn_point_jacobi", self.count, c, _ptr(self.coefA[level]),
                             _ptr(r), _ptr(u), self.omega, st)
        return u

    def vcycle(self, b, level=None):
        """One V-cycle from zero for the batch (multigrid.py:205-222); b (count, nodes)."""
        import torch
        level = self.levels - 1 if level is None else level
        p = self.problem
        st = _native.stream_ptr()
        if level == 0:
            r = b.clone()
            x = torch.empty_like(b)
            _native.call("rbws_fn_band_solve", self.count, p.cells[0], 0, _ptr(self.bands[0]),
                         _ptr(r), _ptr(x), 1.0, 0, st)
            return x
        u = self._smooth(level, torch.zeros_like(b), b, from_zero=True)
        r = self.apply(u, level, b)
        cc = p.cells[level - 1]
        bc = torch.empty(self.count, p.nodes(level - 1), dtype=torch.float64, device="cuda")
        _native.call("rbws_fn_restrict", self.count, cc, _ptr(r), _ptr(bc),
                     _ptr(p._mask_dev[level - 1]), st)
        e = self.vcycle(bc, level - 1)
        _native.call("rbws_fn_prolong_add", self.count, cc, _ptr(e), _ptr(u),
                     _ptr(p._mask_dev[level]), st)
        return self._smooth(level, u, b, forward=False)


def mg_context_for(problem: FnFemProblem, mus, nu: int = 1, smoother: str = "auto"):
    return FnMgContext(problem, mus, nu, smoother)


def mgcg_solve(ctx: FnMgContext, f, x0=None, delta: float = 1e-16, l_max: int = 40,
               method: str = "mgcg"):
    """Batched PCG with one V-cycle per preconditioner application (krylov.py:42-109,
    multigrid.py:225-232): every instance follows the reference's recurrence and stops
    on its own ||r||/||f|| <= delta (finished instances are frozen)."""
    import torch
    if delta <= 0:
        raise ValueError("tolerance must be positive")
    if l_max < 0:
        raise ValueError("l_max must be non-negative")
    t0 = time.perf_counter()
    x = torch.zeros_like(f) if x0 is None else x0.clone()
    fnorm = torch.linalg.vector_norm(f, dim=1)
    absolute = fnorm == 0.0
    scale = torch.where(absolute, torch.ones_like(fnorm), fnorm)
    r = ctx.apply(x, b=f)
    res = torch.linalg.vector_norm(r, dim=1) / scale
    hist = [res]
    active = (res > delta) & (l_max > 0)
    iters = torch.zeros_like(res, dtype=torch.int64)
    if bool(active.any()):
        s = ctx.vcycle(r)
        p = s.clone()
        rs = (r * s).sum(1)
        for k in range(l_max):
            if not bool(active.any()):
                break
            a = active[:, None]
            Ap = ctx.apply(p)
            pAp = (p * Ap).sum(1)
            if bool((pAp[active] <= 0.0).any()):
                raise OperatorError("non-positive curvature p.A.p; operator not SPD")
            alpha = torch.where(active, rs / torch.where(active, pAp, torch.ones_like(pAp)),
                                torch.zeros_like(rs))
            x = torch.where(a, x + alpha[:, None] * p, x)
            r = torch.where(a, r - alpha[:, None] * Ap, r)
            iters = iters + active.to(torch.int64)
            res = torch.where(active, torch.linalg.vector_norm(r, dim=1) / scale, res)
            hist.append(torch.where(active, res, torch.full_like(res, float("nan"))))
            active = active & (res > delta)
            if not bool(active.any()) or k + 1 == l_max:
                break
            s = ctx.vcycle(r)
            rs_new = (r * s).sum(1)
            beta = rs_new / torch.where(active, rs, torch.ones_like(rs))
            p = torch.where(active[:, None], s + beta[:, None] * p, p)
            rs = torch.where(active, rs_new, rs)
    tres = torch.linalg.vector_norm(ctx.apply(x, b=f), dim=1) / scale
    H = torch.stack(hist, 1).cpu().numpy()
    status = np.where(absolute.cpu().numpy(), 4, 0)
    reps = SolveReports(method, iters.cpu().numpy(), H, tres.cpu().numpy(), status,
                        time.perf_counter() - t0, delta, l_max, ctx.mus,
                        {"smoother": ctx.smoother, "layout": "full-node"})
    return x, reps
