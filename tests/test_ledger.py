"""Real-time phase ledger: CostLedger-compatible
accounting of measured GPU time per phase (reference parcost.py:63-122)."""

import os
import sys

import numpy as np
import pytest

from paper_2401_00228_b200.ledger import PhaseLedger, charge_records, phase_of, report_relative

REF = "/root/reference/pkg/src"


def test_charge_attribution_and_fraction():
    led = PhaseLedger(n_proc=2, n_cgs=3)
    led.charge("matvec", [5, 7, 1])            # lanes [6, 7] -> +7
    led.charge("matvec", [4], level=2)         # level >= 1 -> coarse_solve
    led.charge("orthogonalization", [3], parallel=False)
    assert led.phase_elapsed == {"matvec": 7, "coarse_solve": 4, "orthogonalization": 3}
    assert led.elapsed == 14
    assert led.total_work("matvec") == 13 and led.total_work() == 20
    assert led.cgs_fraction() == pytest.approx(4 / 14)
    assert sorted(led.rows())[:2] == [("coarse_solve", 0, 4), ("coarse_solve", 1, 0)]
    with pytest.raises(ValueError):
        led.charge("matvec", [-1])
    with pytest.raises(ValueError):
        PhaseLedger(n_proc=0)


def test_records_to_phases():
    recs = [
        {"level": -1, "hint": None, "category": "march_mv", "ms": 1.0},
        {"level": 0, "hint": None, "category": "march_mvr", "ms": 2.0},
        {"level": 0, "hint": None, "category": "mgs_pass", "ms": 3.0},
        {"level": 0, "hint": "interpolation", "category": "coarse_gemm", "ms": 0.5},
        {"level": 0, "hint": None, "category": "assemble", "ms": 0.25},
        {"level": 1, "hint": None, "category": "march_imv", "ms": 4.0},
        {"level": 3, "hint": None, "category": "coarse_recurrence", "ms": 1.5},
    ]
    assert phase_of(recs[3]) == "interpolation" and phase_of(recs[4]) == "krylov_other"
    led = PhaseLedger()
    charge_records(led, recs)
    assert led.phase_elapsed == {"matvec": 3000, "orthogonalization": 3000,
                                 "interpolation": 500, "krylov_other": 250,
                                 "coarse_solve": 5500}
    assert led.level_ms()[0]["march_mv"] == 1.0
    theta = PhaseLedger()
    theta.charge("theta_scheme", [1000], parallel=False)
    rel = report_relative(led, theta)
    assert rel["relative_total"] == pytest.approx(12.25)
    assert rel["cgs_fraction"] == pytest.approx(5500 / 12250)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_matches_reference_cost_ledger_semantics():
    """Same charges into the reference CostLedger and PhaseLedger give the
    same per-processor work, phase times and CGS fraction."""
    sys.path.insert(0, REF)
    try:
        from pintmk.parcost import CostLedger
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(5)
    a, b = CostLedger(n_proc=3, n_cgs=2), PhaseLedger(n_proc=3, n_cgs=2)
    phases = list(PhaseLedger.PHASES)
    for _ in range(200):
        ph = phases[rng.integers(len(phases))]
        costs = rng.integers(0, 50, rng.integers(1, 9)).tolist()
        par = bool(rng.integers(2))
        lvl = int(rng.integers(0, 3))
        a.charge(ph, costs, parallel=par, level=lvl)
        b.charge(ph, costs, parallel=par, level=lvl)
    assert a.proc_work == b.proc_work
    assert a.phase_elapsed == b.phase_elapsed and a.elapsed == b.elapsed
    assert a.cgs_fraction() == b.cgs_fraction()
    assert sorted(a.rows()) == sorted(b.rows())


@pytest.mark.gpu
def test_solve_with_measured_ledger():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2401_00228_b200 import (PhaseLedger, measured_theta_scheme_ledger,
                                       multilevel_solve, report_relative)
    from tests.cases import SMALL, gpu_hierarchy

    case = SMALL["c5_small"]
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c5_small.npz"))
    h = gpu_hierarchy(case)
    led = PhaseLedger()
    x, rep = multilevel_solve(h, ledger=led)
    assert abs(rep.outer_iterations - int(g["iters"])) <= 1
    assert np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]) <= 1e-10
    for ph in ("matvec", "orthogonalization", "coarse_solve"):
        assert led.phase_elapsed.get(ph, 0) > 0, led.phase_elapsed
    assert 0.0 < led.cgs_fraction() < 1.0
    assert rep.simulated_elapsed == led.elapsed
    # every level of the hierarchy shows up, the coarsest as coarse work
    levels = led.level_ms()
    assert set(levels) == set(range(h.n_levels)), levels
    assert any(c.startswith("coarse") for c in levels[h.n_levels - 1])
    assert sum(rep.metadata["gpu_phase_ms"].values()) == pytest.approx(
        sum(r["ms"] for r in led.records))
    # theta-scheme reference ledger and the relative report
    th = measured_theta_scheme_ledger(h.fine.ops, case.u0_vector())
    assert th.phase_elapsed.get("theta_scheme", 0) > 0
    rel = report_relative(led, th)
    assert rel["relative_total"] > 0 and 0 < rel["cgs_fraction"] < 1
