"""Phase breakdown of bench.py's e2e step (public API, host buffers):
operator build, FineSystem (H2D of u0), hierarchy build, solve, D2H.

    python tools/e2e_timing.py [case] [repeats]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_00228_b200 as P  # noqa: E402
from tests.cases import BASELINE  # noqa: E402


def main():
    case = BASELINE[sys.argv[1] if len(sys.argv) > 1 else "c5_c"]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    pin_u0 = torch.from_numpy(case.u0_vector()).pin_memory()
    pin_x = torch.empty(case.N, dtype=torch.float64).pin_memory()
    for r in range(reps):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        op = P.build_laplacian(case.dim, case.nx, case.ny if case.dim == 2 else 1)
        ops = P.build_step_operators(op, P.ThetaSchemeConfig(case.theta, case.dt(), case.n_t))
        torch.cuda.synchronize(); t.append(time.perf_counter())
        fine = P.FineSystem(ops, pin_u0)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        cfg = P.SolverConfig(mu=case.mu, tol=case.tol, max_outer=case.max_outer,
                             inner_iters=case.inner_iters, coarsest_n_cgs=case.n_cgs,
                             restart=case.restart)
        h = P.build_hierarchy(fine, case.n_levels, list(case.schedule), cfg, nu=case.nu)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        x, rep = P.multilevel_solve(h, out=pin_x)  # x streamed to pinned memory
        torch.cuda.synchronize(); t.append(time.perf_counter())
        names = ["operators", "FineSystem(H2D u0)", "build_hierarchy", "solve + D2H x"]
        d = {n: 1e3 * (t[i + 1] - t[i]) for i, n in enumerate(names)}
        print(f"rep {r}: total {1e3 * (t[-1] - t[0]):.1f} ms  " +
              "  ".join(f"{n} {v:.1f}" for n, v in d.items()), flush=True)
        del h, fine, x
        gb = 1e-9
        a0, r0 = torch.cuda.memory_allocated() * gb, torch.cuda.memory_reserved() * gb
        if os.environ.get("E2E_GC"):
            import gc
            gc.collect()
        print(f"   after del: allocated {a0:.1f} GB reserved {r0:.1f} GB; after gc: "
              f"allocated {torch.cuda.memory_allocated() * gb:.1f} GB", flush=True)


if __name__ == "__main__":
    main()
