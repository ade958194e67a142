"""B200-native all-at-once space-time MLK solve (arXiv 2401.00228).

Drop-in for the reference package ``pintmk``'s solver path: the same
setup/solve API (build_laplacian -> ThetaSchemeConfig -> build_step_operators
-> FineSystem -> build_hierarchy -> multilevel_solve), with every space-time
vector operation running in hand-written sm_100a kernels
(``libpmk_b200.so``, C-ABI in ``include/pintmk_b200.h``).
"""

from .spatial import (SpatialOperator, build_laplacian, courant_number,  # noqa: F401
                      delta_t_for_courant, gershgorin_bound, initial_bump,
                      max_eigenvalue_magnitude)
from .stepper import (BlockBidiagonalSystem, FineSystem, StepOperators,  # noqa: F401
                      ThetaSchemeConfig, build_step_operators, sequential_solve)
from .intergrid import (CoarseSystem, MgritPair, TimePair, TimeSpacePair, WeightedSpacePair,  # noqa: F401
                        agglomerate_partition, perturb_decouple, rediscretized_coarse)
from .solver import (Level, LevelHierarchy, SolveReport, SolverConfig,  # noqa: F401
                     apply_preconditioner, build_hierarchy, build_two_level, fgmres,
                     multilevel_solve, two_level_solve)

from .ledger import (PhaseLedger, measured_theta_scheme_ledger,  # noqa: F401
                     report_relative)

__version__ = "0.1.0"
