"""Solve reports and errors of the batched Krylov path.

Mirrors reference krylov.py:21-39 (OperatorError, SolveReport).  The
batched PCG itself is native (rbws_mgcg_solve, csrc/solver.cu); the Python
entry point is ``multigrid.mgcg_solve`` / ``krylov.pcg_solve``.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np


class OperatorError(Exception):
    """The operator violated the SPD contract (breakdown, zero diagonal...)."""


@dataclass
class SolveReport:
    """Convergence record of one iterative solve (krylov.py:25-39)."""

    method: str
    iterations: int
    history: list  # relative recurrence residuals, length iterations+1
    converged: bool
    true_residual: float  # recomputed ||f - A x|| / ||f|| at exit
    wall_time: float
    delta: float
    l_max: int
    mu: np.ndarray | None = None
    absolute_norms: bool = False
    config: dict = field(default_factory=dict)


class SolveReports(Sequence):
    """The SolveReport list of one batched solve, materialised lazily.

    Holds the per-instance arrays the native solver returned; ``reports[m]`` builds
    (and caches) instance m's SolveReport.  Building 1024 report objects costs
    milliseconds of host time, during which the GPU would idle between batches.
    ``iterations`` / ``true_residuals`` / ``converged`` give vectorised access.
    """

    def __init__(self, method, iters, hist, tres, status, wall, delta, l_max, mus, config):
        self.method, self.delta, self.l_max = method, delta, l_max
        self.iterations = np.asarray(iters)
        self._hist, self.true_residuals = hist, np.asarray(tres)
        self._status, self._wall, self._mus = np.asarray(status), wall, mus
        self._config = dict(config)
        self._cache = {}

    @property
    def converged(self):
        return self.true_residuals <= self.delta

    def update_config(self, **kw):
        self._config.update(kw)
        for r in self._cache.values():
            r.config.update(kw)

    def __len__(self):
        return len(self.iterations)

    def __getitem__(self, m):
        if isinstance(m, slice):
            return [self[i] for i in range(*m.indices(len(self)))]
        if m < 0:
            m += len(self)
        if not 0 <= m < len(self):
            raise IndexError(m)
        r = self._cache.get(m)
        if r is None:
            k = int(self.iterations[m])
            r = SolveReport(
                method=self.method, iterations=k,
                history=[float(v) for v in self._hist[m, :k + 1]],
                converged=bool(self.true_residuals[m] <= self.delta),
                true_residual=float(self.true_residuals[m]),
                wall_time=self._wall / len(self), delta=self.delta, l_max=self.l_max,
                mu=None if self._mus is None else np.asarray(self._mus[m]),
                absolute_norms=bool(self._status[m] & 4), config=dict(self._config))
            self._cache[m] = r
        return r

    @classmethod
    def concat(cls, parts):
        """One lazy sequence over several batches (same method / tolerance)."""
        parts = [p for p in parts if len(p)]
        if not parts:
            return []
        p0 = parts[0]
        L = max(p._hist.shape[1] for p in parts)
        hist = np.full((sum(len(p) for p in parts), L), np.nan)
        o = 0
        for p in parts:
            hist[o:o + len(p), :p._hist.shape[1]] = p._hist
            o += len(p)
        mus = None if p0._mus is None else np.concatenate([np.asarray(p._mus) for p in parts])
        out = cls(p0.method, np.concatenate([p.iterations for p in parts]), hist,
                  np.concatenate([p.true_residuals for p in parts]),
                  np.concatenate([p._status for p in parts]),
                  sum(p._wall for p in parts), p0.delta, p0.l_max, mus, p0._config)
        return out


def pcg_solve(A, f, x0, precond=None, delta: float = 1e-16, l_max: int = 40,
              method: str = "pcg", mu=None):
    """Batched PCG (krylov.py:42-109) with the multigrid preconditioner.

    ``precond`` must be the batch's MgContext (the B200 path fuses the
    preconditioner into the native PCG loop); A is the BatchOperator bound
    to the same context.
    """
    from .multigrid import MgContext, mgcg_solve
    if not isinstance(precond, MgContext):
        raise ValueError("the B200 PCG path takes the batch MgContext as preconditioner")
    return mgcg_solve(A, f, x0, precond, delta=delta, l_max=l_max, mu=mu, method=method)
