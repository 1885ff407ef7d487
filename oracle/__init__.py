"""CPU oracle for the RBWS hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference algorithms
(``/root/reference/pkg/src/rbws``) on the data-parallel path this repo
accelerates: parametrised diffusion operators on nested grids, Galerkin
coarsening, the damped-Jacobi V-cycle, preconditioned CG, and the L1ROC
over-collocation reduced model (online least squares + offline greedy with
DEIM).  Every function cites the reference file:line it restates.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or the timed CPU baseline — never as part of the product path
(``paper_2311_13862_b200`` never imports it).

Parity pin: ``tests/golden/make_golden.py`` runs the real reference package
(built from ``/root/reference`` into /tmp, Cython backend) on the same
inputs and commits its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py``
checks this restatement against them.
"""

from .problems import (FDProblemSpec, OracleProblem, sample_mus, smooth_affine,
                       thermal_block)
from .solvers import (OracleMgContext, SolveReport, deim_extend, galerkin,
                      jacobi_sweep, l1_indicator, l1roc_offline, l1roc_online,
                      lhs_sample, mg_context_for, mg_vcycle, mgcg_solve,
                      pcg_solve, rbi_mgcg_solve)

__all__ = [
    "FDProblemSpec", "OracleProblem", "sample_mus", "smooth_affine",
    "thermal_block", "OracleMgContext", "SolveReport", "deim_extend",
    "galerkin", "jacobi_sweep", "l1_indicator", "l1roc_offline",
    "l1roc_online", "lhs_sample", "mg_context_for", "mg_vcycle",
    "mgcg_solve", "pcg_solve", "rbi_mgcg_solve",
]
