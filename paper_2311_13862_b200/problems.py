"""Parametrised diffusion problems of the BASELINE configurations.

Mirrors the reference's ``ProblemSpec`` (reference problems.py:26-75):
a parameter box, affine diffusion terms ``K(x; mu) = sum_q theta_q(mu) k_q(x)``
and a source.  Here every term is *separable along the grid axes*, which is
what lets the B200 path keep the finest operator implicit: each term is
described by 1D factor tables (see include/rbws_b200.h) instead of an
assembled sparse matrix.

Discretisation: vertex-centred finite volumes on n cells per
axis, homogeneous Dirichlet boundary, edge weight = h * (mean of the term's
coefficient over the dual face), rhs = h^3 f at interior nodes.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ProblemSpec:
    """A parametrised FV diffusion problem on the unit cube."""

    pid: str
    kind: str                      # "thermal-block" | "smooth-affine"
    p: int
    bounds: tuple                  # ((lo, hi),) * p
    blocks: tuple = (1, 1, 1)
    sampling: str = "log-uniform"
    n_modes: int = 0

    @property
    def n_terms(self) -> int:
        return self.p if self.kind == "thermal-block" else self.n_modes + 1

    def check_mu(self, mu) -> np.ndarray:
        """Validate one parameter (reference problems.py:47-53)."""
        mu = np.asarray(mu, dtype=np.float64)
        if mu.shape != (self.p,):
            raise ValueError(f"{self.pid} expects {self.p}-dimensional parameters")
        b = np.asarray(self.bounds, dtype=np.float64)
        if np.any(mu < b[:, 0]) or np.any(mu > b[:, 1]):
            raise ValueError(f"parameter {mu} outside {self.pid} bounds")
        return mu

    def check_mus(self, mus) -> np.ndarray:
        mus = np.atleast_2d(np.asarray(mus, dtype=np.float64))
        if mus.shape[1] != self.p:
            raise ValueError(f"{self.pid} expects {self.p}-dimensional parameters")
        b = np.asarray(self.bounds, dtype=np.float64)
        if np.any(mus < b[:, 0]) or np.any(mus > b[:, 1]):
            raise ValueError(f"parameters outside {self.pid} bounds")
        return mus

    def thetas(self, mus) -> np.ndarray:
        """theta_q(mu) for a batch, shape (count, Q)."""
        mus = self.check_mus(mus)
        if self.kind == "thermal-block":
            return mus.copy()
        return np.concatenate([np.ones((len(mus), 1)), mus], axis=1)

    # ------------------------------------------------------------ tables
    def separable_tables(self, n: int):
        """(face[Q,3,n], node[Q,3,3,n+1]) for an n-cell grid."""
        Q = self.n_terms
        face = np.zeros((Q, 3, n))
        node = np.zeros((Q, 3, 3, n + 1))
        h = 1.0 / n
        if self.kind == "thermal-block":
            nb = self.blocks
            if any(n % b for b in nb):
                raise ValueError("block interfaces must fall on grid planes")
            for q in range(Q):
                cell = (q % nb[0], (q // nb[0]) % nb[1], q // (nb[0] * nb[1]))
                for d in range(3):
                    for a in range(3):
                        s = cell[a] * n // nb[a]
                        e = (cell[a] + 1) * n // nb[a]
                        if a == d:
                            face[q, d, s:e] = h
                        else:
                            frac = np.zeros(n + 1)
                            frac[s + 1:e] = 1.0
                            frac[s] = 0.5
                            frac[e] = 0.5
                            node[q, d, a] = frac
        else:
            xf = (np.arange(n) + 0.5) * h
            xn = np.arange(n + 1) * h
            for q in range(Q):
                for d in range(3):
                    if q == 0:
                        face[q, d] = h
                        for a in range(3):
                            if a != d:
                                node[q, d, a] = 1.0
                        continue
                    k = q
                    g = (lambda t: np.sin(k * np.pi * t), lambda t: np.sin(k * np.pi * t),
                         lambda t: np.cos(k * np.pi * t))
                    face[q, d] = h * g[d](xf)
                    for a in range(3):
                        if a != d:
                            node[q, d, a] = g[a](xn)
        return face, node

    def rhs_padded(self, n: int, device="cuda"):
        """h^3 f(X) in the padded single-instance layout (n^3 + n^2 doubles)."""
        import torch
        h = 1.0 / n
        out = torch.zeros(n * n * n + 2 * n * n, dtype=torch.float64, device=device)
        idx = torch.arange(n, dtype=torch.float64, device=device) * h
        if self.kind == "thermal-block":
            f = torch.ones((n, n, n), dtype=torch.float64, device=device)
        else:
            g = torch.exp(-((idx - 0.5) ** 2) / 0.02)
            f = g[:, None, None] * g[None, :, None] * g[None, None, :]
        f = h ** 3 * f
        f[0, :, :] = 0.0
        f[:, 0, :] = 0.0
        f[:, :, 0] = 0.0
        out[: n ** 3] = f.reshape(-1)
        return out


def thermal_block(blocks=(2, 1, 1)) -> ProblemSpec:
    bx, by, bz = blocks
    p = bx * by * bz
    return ProblemSpec(pid=f"thermal-block-{bx}x{by}x{bz}", kind="thermal-block", p=p,
                       bounds=((0.1, 10.0),) * p, blocks=(bx, by, bz), sampling="log-uniform")


def smooth_affine(n_modes: int = 6) -> ProblemSpec:
    return ProblemSpec(pid=f"smooth-affine-{n_modes}", kind="smooth-affine", p=n_modes,
                       bounds=((-0.1, 0.1),) * n_modes, sampling="uniform", n_modes=n_modes)


_REGISTRY = {
    "thermal-block-2x1x1": lambda: thermal_block((2, 1, 1)),
    "thermal-block-2x2x1": lambda: thermal_block((2, 2, 1)),
    "thermal-block-2x2x2": lambda: thermal_block((2, 2, 2)),
    "smooth-affine-6": lambda: smooth_affine(6),
}


def _fem(name):
    def make():
        from . import fem
        return getattr(fem, name)()
    return make


# the reference's own assembled (Q1 FEM) problems, problems.py:96-155
_REGISTRY["example-1"] = _fem("example1")
_REGISTRY["example-2"] = _fem("example2")


def get_problem(pid: str):
    """Registry lookup (reference problems.py:158-162)."""
    try:
        return _REGISTRY[pid]()
    except KeyError:
        raise ValueError(f"unknown problem id {pid!r}; choices: {sorted(_REGISTRY)}") from None


def sample_mus(spec: ProblemSpec, count: int, seed: int) -> np.ndarray:
    """BASELINE sampling: log-uniform in the box or uniform (seeded)."""
    rng = np.random.default_rng(seed)
    b = np.asarray(spec.bounds, dtype=np.float64)
    u = rng.random((count, spec.p))
    if spec.sampling == "log-uniform":
        lo, hi = np.log(b[:, 0]), np.log(b[:, 1])
        return np.exp(lo + u * (hi - lo))
    return b[:, 0] + u * (b[:, 1] - b[:, 0])


def lhs_sample(p: int, n: int, bounds, seed: int = 0) -> list:
    """Seeded Latin hypercube over a box (the reference's sampling, sampling.py:8-27): one
    point per stratum per axis, generator draws the in-stratum offsets then one permutation
    per axis."""
    if n < 1:
        raise ValueError("need at least one sample")
    b = np.asarray(bounds, dtype=np.float64)
    if b.shape != (p, 2):
        raise ValueError(f"bounds must be ({p}, 2), got {b.shape}")
    if np.any(b[:, 1] <= b[:, 0]):
        raise ValueError("degenerate bounds: need min < max per dimension")
    g = np.random.default_rng(seed)
    offsets = g.random((n, p))
    strata = np.column_stack([g.permutation(n) for _ in range(p)])
    u = (offsets + strata) / n
    pts = b[:, 0] + u * (b[:, 1] - b[:, 0])
    return [row.copy() for row in pts]


def levels_for(n: int, m0: int) -> int:
    r = n // m0
    if n % m0 or r & (r - 1):
        raise ValueError("n must be m0 * 2^J")
    return int(math.log2(r)) + 1
