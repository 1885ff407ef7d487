"""Nested grids, padded device layout and the batched parametric operator.

B200 counterpart of the reference ``grid.py`` (ParametricProblem,
grid.py:193-290; build_hierarchy, grid.py:163-170).  The reference assembles
sparse matrices per term and Galerkin-coarsens them with scipy; here the
mu-independent part (the hierarchy and the Kronecker factors of every term
on every level) lives in the native ``rbws_hierarchy`` and per-parameter
operators only ever exist on the device, batched.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .problems import ProblemSpec, levels_for


def padded_len(n: int, count: int) -> int:
    """Doubles in a padded batch vector of `count` instances on n cells."""
    return count * n ** 3 + 2 * n * n


def to_padded(v, n: int, device="cuda"):
    """Interior-ordered vectors (count, (n-1)^3) or ((n-1)^3,) -> padded batch tensor."""
    import torch
    a = torch.as_tensor(np.asarray(v, dtype=np.float64))
    if a.dim() == 1:
        a = a[None]
    count, m = a.shape[0], n - 1
    if a.shape[1] != m ** 3:
        raise ValueError("vector length does not match the grid's free DoFs")
    out = torch.zeros(padded_len(n, count), dtype=torch.float64, device=device)
    blk = out[: count * n ** 3].view(count, n, n, n)
    blk[:, 1:, 1:, 1:] = a.view(count, m, m, m).to(device)
    return out


def from_padded(x, n: int, count: int) -> np.ndarray:
    """Padded batch tensor -> numpy (count, (n-1)^3) in the reference's free-DoF order."""
    blk = x[: count * n ** 3].view(count, n, n, n)[:, 1:, 1:, 1:]
    return blk.reshape(count, -1).cpu().numpy()


def interior_to_padded_index(idx, n: int) -> np.ndarray:
    """Free-DoF indices (reference ordering) -> padded node indices."""
    idx = np.asarray(idx, dtype=np.int64)
    m = n - 1
    i, j, k = idx % m + 1, (idx // m) % m + 1, idx // (m * m) + 1
    return i + n * (j + n * k)


def padded_to_interior_index(pidx, n: int) -> np.ndarray:
    pidx = np.asarray(pidx, dtype=np.int64)
    m = n - 1
    i, j, k = pidx % n - 1, (pidx // n) % n - 1, pidx // (n * n) - 1
    return i + m * (j + m * k)


class ParametricProblem:
    """Factory for batched A_h(mu), f_h(mu) and the multigrid hierarchy.

    Signature mirrors the reference (grid.py:203): ``levels`` nested grids of
    ``m0 * 2**i`` cells.  Immutable after construction.
    """

    def __new__(cls, spec, levels: int = 3, m0: int = 2):
        if getattr(spec, "kind", None) == "fem":  # assembled problems (fem.py)
            if spec.neumann_face_x1:  # free boundary nodes: full-node layout (fem_fn.py)
                from .fem_fn import FnFemProblem
                return FnFemProblem(spec, levels, m0)
            from .fem import FemProblem
            return FemProblem(spec, levels, m0)
        return super().__new__(cls)

    def __init__(self, spec: ProblemSpec, levels: int = 3, m0: int = 2):
        if levels < 2:
            raise ValueError("need at least 2 levels for coarse-grid correction")
        if m0 < 2:
            raise ValueError("base grid needs at least 2 cells per dimension")
        _native.require_cuda()
        self.spec = spec
        self.m0 = m0
        self.cells = tuple(m0 * 2 ** i for i in range(levels))
        self.n = self.cells[-1]
        self.n_free = (self.n - 1) ** 3
        self.face, self.node = spec.separable_tables(self.n)
        h = ctypes.c_void_p()
        _native.call("rbws_hierarchy_create", ctypes.byref(h), self.n, m0, spec.n_terms,
                     self.face.ctypes.data, self.node.ctypes.data)
        self._h = h
        self._rhs = spec.rhs_padded(self.n)

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

    def factors(self, level: int) -> np.ndarray:
        """1D Kronecker factors of every term on `level`: [Q,3(part),3(axis),2,n+1]."""
        n = self.cells[level]
        Q = self.spec.n_terms
        out = np.zeros((Q, 3, 3, 2, n + 1))
        _native.call("rbws_hierarchy_factors", self._h, level, out.ctypes.data, out.size)
        return out

    def thetas(self, mus):
        import torch
        return torch.as_tensor(self.spec.thetas(mus), dtype=torch.float64, device="cuda")

    def rhs(self, mu=None):
        """f_h (shared by all mu for these problems): padded single-instance vector."""
        if mu is not None:
            self.spec.check_mus(mu)
        return self._rhs

    def zeros(self, count: int, level: int | None = None):
        import torch
        n = self.cells[self.finest_level if level is None else level]
        return torch.zeros(padded_len(n, count), dtype=torch.float64, device="cuda")

    def operator(self, mus, ctx=None):
        """Batched operator A_h(mu) for the given parameters (grid.py:246-255)."""
        from .multigrid import mg_context_for
        if ctx is None:
            ctx = mg_context_for(self, mus)
        return BatchOperator(ctx)


class BatchOperator:
    """A_h(mu) for a batch, bound to an MgContext; ``A @ x`` on padded tensors."""

    def __init__(self, ctx):
        self.ctx = ctx

    @property
    def count(self):
        return self.ctx.count

    def apply(self, x, level: int | None = None):
        import torch
        prob = self.ctx.problem
        lvl = prob.finest_level if level is None else level
        y = torch.zeros_like(x)
        _native.call("rbws_apply", self.ctx.handle, lvl, x.data_ptr(), y.data_ptr(),
                     _native.stream_ptr())
        return y

    def __matmul__(self, x):
        return self.apply(x)
