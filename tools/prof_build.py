"""cProfile of the e2e setup path (operators, FineSystem, build_hierarchy) for
one case, after a warm-up build.

    python tools/prof_build.py [case] [n_lines]
"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_00228_b200 as P  # noqa: E402
from tests.cases import BASELINE  # noqa: E402

case = BASELINE[sys.argv[1] if len(sys.argv) > 1 else "c5_c"]
pin_u0 = torch.from_numpy(case.u0_vector()).pin_memory()


def build():
    op = P.build_laplacian(case.dim, case.nx, case.ny if case.dim == 2 else 1)
    ops = P.build_step_operators(op, P.ThetaSchemeConfig(case.theta, case.dt(), case.n_t))
    fine = P.FineSystem(ops, pin_u0)
    cfg = P.SolverConfig(mu=case.mu, tol=case.tol, max_outer=case.max_outer,
                         coarsest_n_cgs=case.n_cgs, restart=case.restart)
    h = P.build_hierarchy(fine, case.n_levels, list(case.schedule), cfg, nu=case.nu)
    torch.cuda.synchronize()
    return h


h = build()
del h
pr = cProfile.Profile()
pr.enable()
h = build()
pr.disable()
pstats.Stats(pr).sort_stats(os.environ.get("PROF_SORT", "tottime")).print_stats(
    int(sys.argv[2]) if len(sys.argv) > 2 else 25)
