"""Solve reports and errors of the batched Krylov path.

Mirrors reference krylov.py:246-264 (OperatorError, SolveReport).  The
batched PCG itself is native (rbws_mgcg_solve, csrc/solver.cu); the Python
entry point is ``multigrid.mgcg_solve`` / ``krylov.pcg_solve``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class OperatorError(Exception):
    """The operator violated the SPD contract (breakdown, zero diagonal...)."""


@dataclass
class SolveReport:
    """Convergence record of one iterative solve (krylov.py:250-264)."""

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


def pcg_solve(A, f, x0, precond=None, delta: float = 1e-16, l_max: int = 40,
              method: str = "pcg", mu=None):
    """Batched PCG (krylov.py:267-334) with the multigrid preconditioner.

    ``precond`` must be the batch's MgContext (the B200 path fuses the
    preconditioner into the native PCG loop); A is the BatchOperator bound
    to the same context.
    """
    from .multigrid import MgContext, mgcg_solve
    if not isinstance(precond, MgContext):
        raise ValueError("the B200 PCG path takes the batch MgContext as preconditioner")
    return mgcg_solve(A, f, x0, precond, delta=delta, l_max=l_max, mu=mu, method=method)
