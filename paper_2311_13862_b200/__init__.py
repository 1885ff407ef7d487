"""B200-native reduced-basis warm-started MGCG (the RBWS hot path).

Drop-in, batched counterpart of the reference package ``rbws`` on the
MGCG / RBI-MGCG path: problems, grid hierarchy, multigrid context, V-cycle,
PCG, and the L1ROC over-collocation model (online + greedy offline), all
running through the C ABI in include/rbws_b200.h (sm_100a CUDA kernels).
"""

from .grid import (BatchOperator, ParametricProblem, from_padded, padded_len,
                   to_padded)
from .hf import HighFidelitySolver
from .krylov import OperatorError, SolveReport, pcg_solve
from .multigrid import MgContext, mg_context_for, mg_vcycle, mgcg_solve
from .msrb import MsrbHierarchy, PodBasis, msrb_train, pod_build, rbi_msrbcg_solve
from .pipeline import HostPipeline
from .problems import (ProblemSpec, get_problem, lhs_sample, sample_mus, smooth_affine,
                       thermal_block)
from .slab import SlabSolver, slab_mgcg_solve, slab_partition
from .rb import (DegenerateBasisError, L1rocModel, deim_extend, l1_indicator,
                 l1roc_offline, l1roc_online)
from .warmstart import (METHODS, MethodConfig, initial_residual,
                        make_initial_guess, rbi_pcg_solve)

__version__ = "0.1.0"
