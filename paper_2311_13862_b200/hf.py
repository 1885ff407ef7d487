"""High-fidelity solves for snapshot generation (reference hf.py:12-60).

The reference factors A_h(mu) with SuperLU; on the B200 the high-fidelity
solve is the batched MGCG driven to a tight tolerance (the reference's
``method="mgcg"`` branch, hf.py:40-57, delta=1e-14, l_max=100).
"""

from __future__ import annotations

import numpy as np

from .grid import ParametricProblem
from .multigrid import mg_context_for, mgcg_solve


class HighFidelitySolver:
    def __init__(self, problem: ParametricProblem, method: str = "mgcg", delta: float = 1e-14,
                 l_max: int = 100, nu: int = 1, smoother: str = "auto"):
        if method != "mgcg":
            raise ValueError("the B200 high-fidelity solver is MGCG (no sparse LU on device)")
        self.problem = problem
        self.method = method
        self.delta = delta
        self.l_max = l_max
        self.nu = nu
        self.smoother = smoother
        self._ctx = None
        self.last_reports = None

    def solve_batch(self, mus, rhs=None):
        """Solutions for a batch of parameters (padded device tensor)."""
        mus = self.problem.spec.check_mus(mus)
        self._ctx = mg_context_for(self.problem, mus, nu=self.nu, smoother=self.smoother,
                                   ctx=self._ctx)
        f = self.problem.rhs(mus) if rhs is None else rhs
        x, reps = mgcg_solve(None, f, None, self._ctx, delta=self.delta, l_max=self.l_max)
        self.last_reports = reps
        return x

    def solve(self, mu, rhs=None):
        return self.solve_batch(np.asarray(mu, dtype=np.float64)[None], rhs)

    def __call__(self, mu, rhs=None):
        return self.solve(mu, rhs)
