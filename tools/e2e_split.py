"""Split one e2e step of the c5_c workload into host setup, hierarchy upload,
solve and result copy (wall clock with device syncs between phases)."""
import os, sys, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_00228_b200 as P
from tests.cases import BASELINE as CASES

case = CASES["c5_c"]
pin_u0 = torch.from_numpy(case.u0_vector()).pin_memory()
pin_x = torch.empty(case.N, dtype=torch.float64).pin_memory()


def step(report):
    s = torch.cuda.synchronize
    s(); t = [time.perf_counter()]
    op = P.build_laplacian(case.dim, case.nx, case.ny)
    ops = P.build_step_operators(op, P.ThetaSchemeConfig(case.theta, case.dt(), case.n_t))
    s(); t.append(time.perf_counter())
    fine = P.FineSystem(ops, pin_u0)
    s(); t.append(time.perf_counter())
    cfg = P.SolverConfig(mu=case.mu, tol=case.tol, max_outer=case.max_outer,
                         inner_iters=case.inner_iters, coarsest_n_cgs=case.n_cgs,
                         restart=case.restart)
    h = P.build_hierarchy(fine, case.n_levels, list(case.schedule), cfg, nu=case.nu)
    s(); t.append(time.perf_counter())
    x, rep = P.multilevel_solve(h, out=pin_x)
    s(); t.append(time.perf_counter())
    del h, x, fine
    gc.collect()
    s(); t.append(time.perf_counter())
    if report:
        names = ["laplacian+step_ops", "FineSystem", "build_hierarchy", "solve+D2H", "teardown"]
        print({n: round(1000 * (b - a), 2) for n, a, b in zip(names, t, t[1:])},
              "total", round(1000 * (t[-2] - t[0]), 1), "ms")


for i in range(4):
    step(i >= 2)
