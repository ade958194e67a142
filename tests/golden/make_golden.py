"""Generate golden fixtures from the LIVE reference package (run here, in the
container that has /root/reference; the fixtures travel, the reference does
not).

    python tests/golden/make_golden.py [names]        # small cases (full vectors)
    python tests/golden/make_golden.py --mid [names]  # mid cases (fingerprints)

For each small case in tests/cases.py it builds the hierarchy with the
reference's own public API (solver.build_hierarchy / build_two_level; the
"time_space" move through the reference's _space_move(level, time_nu),
solver.py:127-143) and records, from seeded inputs:
  matvec of level 0, restrict/interpolate and apply_preconditioner of every
  non-coarsest level, the coarsest forward_solve, and the full solve
  (iterations, residual history, x, true residual).
Restart cases use the restart wrapper of SURVEY.md section 8(c) around the
reference's fgmres.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

from pintmk import intergrid as R_ig  # noqa: E402
from pintmk import solver as R_sol  # noqa: E402
from pintmk import spatial as R_sp  # noqa: E402
from pintmk import stepper as R_st  # noqa: E402

from tests.cases import SMALL  # noqa: E402


def reference_hierarchy(case):
    op = R_sp.build_laplacian(case.dim, case.nx, case.ny if case.dim == 2 else 1)
    if case.perturb is not None:
        op = R_sp.SpatialOperator(op.dim, op.n_x, op.n_y, op.delta_x, op.tau,
                                  case.spatial_matrix(op.matrix))
    ops = R_st.build_step_operators(op, R_st.ThetaSchemeConfig(case.theta, case.dt(), case.n_t))
    fine = R_st.FineSystem(ops, case.u0_vector(), forcing=case.forcing_array())
    cfg = R_sol.SolverConfig(mu=case.mu, tol=case.tol, max_outer=case.max_outer,
                             inner_iters=case.inner_iters, coarsest_n_cgs=case.n_cgs)
    if case.two_level_family is not None:
        return R_sol.build_two_level(fine, case.two_level_family, case.nu, cfg)
    if case.schedule == "auto" or "time_space" not in case.schedule:
        return R_sol.build_hierarchy(fine, case.n_levels, case.schedule_arg(), cfg, nu=case.nu)
    levels = [R_sol._fine_level(fine)]
    for mv in case.schedule:
        if mv == "time":
            levels.append(R_sol._time_move(levels[-1], case.nu))
        elif mv == "space":
            levels.append(R_sol._space_move(levels[-1]))
        else:
            levels.append(R_sol._space_move(levels[-1], time_nu=case.nu))
    R_sol._assign_budgets(levels, cfg.inner_iters)
    if cfg.coarsest_n_cgs >= 1:
        levels[-1].system = R_ig.perturb_decouple(levels[-1].system, cfg.coarsest_n_cgs)
    levels[-1].system.diag_factorization
    hier = R_sol.LevelHierarchy(levels=levels, fine=fine, config=cfg)
    hier.moves = list(case.schedule)
    return hier


def reference_restarted(hier, tol, max_outer, restart):
    b = hier.fine.rhs.ravel()
    beta0 = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    r = b.copy()
    hist, total = [], 0
    while total < max_outer:
        rn = float(np.linalg.norm(r))
        if rn == 0.0:
            break
        m = min(restart, max_outer - total)
        dx, rep = R_sol.fgmres(hier, 0, r, tol=tol * beta0 / rn, max_iter=m)
        x = x + dx
        total += rep.outer_iterations
        hist += [v * rn / beta0 for v in rep.residual_history]
        r = b - hier.fine.matvec(x)
        if float(np.linalg.norm(r)) / beta0 <= tol:
            break
        if rep.outer_iterations == 0:
            break
    return x, total, hist


def record(case) -> dict:
    hier = reference_hierarchy(case)
    rng = np.random.default_rng(1234)
    out = {"u0": case.u0_vector()}
    lv = hier.levels
    v0 = rng.standard_normal(lv[0].total_dim)
    out["mv_in"] = v0
    out["mv_out"] = lv[0].system.matvec(v0)
    for i in range(len(lv) - 1):
        vi = rng.standard_normal(lv[i].total_dim)
        out[f"r{i}_in"] = vi
        out[f"r{i}_out"] = lv[i].pair.restrict(vi)
        wi = rng.standard_normal(lv[i + 1].total_dim)
        out[f"i{i}_in"] = wi
        out[f"i{i}_out"] = lv[i].pair.interpolate(wi)
    pv = rng.standard_normal(lv[0].total_dim)
    out["pc_in"] = pv
    out["pc_out"] = R_sol.apply_preconditioner(hier, 0, pv)
    cr = rng.standard_normal(lv[-1].total_dim)
    out["cs_in"] = cr
    out["cs_out"] = lv[-1].system.forward_solve(cr)
    if case.restart is None:
        x, rep = R_sol.multilevel_solve(hier)
        out["iters"] = np.array(rep.outer_iterations)
        out["hist"] = np.array(rep.residual_history)
    else:
        x, total, hist = reference_restarted(hier, case.tol, case.max_outer, case.restart)
        out["iters"] = np.array(total)
        out["hist"] = np.array(hist)
    out["x"] = x
    out["true_res"] = np.array(hier.fine.relative_residual(x))
    return out


from tests.cases import MID_STRIDE, fingerprint, mid_inputs  # noqa: E402


def record_mid(case) -> dict:
    """Fingerprints only (the vectors are too large to commit): the
    coarsest forward_solve and apply_preconditioner of seeded inputs, and the
    full solve (iterations, history, true residual, x)."""
    hier = reference_hierarchy(case)
    lv = hier.levels
    cs_in, pc_in = mid_inputs(case, (lv[-1].total_dim, lv[0].total_dim))
    out = {"u0": case.u0_vector(), "stride": np.array(MID_STRIDE)}
    cs = lv[-1].system.forward_solve(cs_in)
    f = fingerprint(cs, lv[-1].n_steps + 1)
    out["cs_sub"], out["cs_norms"] = f["sub"], f["norms"]
    pc = R_sol.apply_preconditioner(hier, 0, pc_in)
    f = fingerprint(pc, lv[0].n_steps + 1)
    out["pc_sub"], out["pc_norms"] = f["sub"], f["norms"]
    x, rep = R_sol.multilevel_solve(hier)
    out["iters"] = np.array(rep.outer_iterations)
    out["hist"] = np.array(rep.residual_history)
    f = fingerprint(x, lv[0].n_steps + 1)
    out["x_sub"], out["x_norms"] = f["sub"], f["norms"]
    out["true_res"] = np.array(hier.fine.relative_residual(x))
    out["moves"] = np.array(hier.moves)
    return out


def main(names=None):
    if names and names[0] == "--mid":
        from tests.cases import MID

        for name, case in MID.items():
            if len(names) > 1 and name not in names[1:]:
                continue
            data = record_mid(case)
            path = os.path.join(HERE, f"{name}.npz")
            np.savez_compressed(path, **data)
            print(f"{name}: iters={int(data['iters'])} true_res={float(data['true_res']):.3e} "
                  f"-> {os.path.getsize(path) / 1024:.0f} KiB", flush=True)
        return
    for name, case in SMALL.items():
        if names and name not in names:
            continue
        data = record(case)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{name}: iters={int(data['iters'])} true_res={float(data['true_res']):.3e} "
              f"-> {os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
