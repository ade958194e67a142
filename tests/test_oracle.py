"""The CPU oracle against the reference: committed golden fixtures (always)
and the live reference (when /root/reference is mounted).  CPU only."""

import os

import numpy as np
import pytest

from oracle import pintmk_oracle as O
from tests.cases import SMALL, oracle_hierarchy

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def oracle_record(case):
    h = oracle_hierarchy(case)
    g = golden(case.name)
    out = {}
    r = h.rungs
    out["mv_out"] = O.matvec(r[0].system, g["mv_in"])
    for i in range(len(r) - 1):
        out[f"r{i}_out"] = O.restrict(r[i].pair, g[f"r{i}_in"])
        out[f"i{i}_out"] = O.interpolate(r[i].pair, g[f"i{i}_in"])
    out["pc_out"] = O.precondition(h, 0, g["pc_in"])
    out["cs_out"] = O.forward_solve(r[-1].system, g["cs_in"])
    x, info = O.solve(h)
    out["x"] = x
    out["iters"] = info["iterations"]
    out["hist"] = np.array(info["history"])
    out["true_res"] = info["true_relative_residual"]
    return out


@pytest.mark.parametrize("name", sorted(SMALL))
def test_oracle_matches_golden_bitwise(name):
    case = SMALL[name]
    g = golden(name)
    np.testing.assert_array_equal(g["u0"], case.u0_vector())
    o = oracle_record(case)
    for key, val in o.items():
        ref = g[key]
        if key == "iters":
            assert int(val) == int(ref)
        else:
            np.testing.assert_array_equal(np.asarray(val), ref, err_msg=f"{name}:{key}")


def test_decouple_dropped_sets():
    # n_T = 8
    assert O.decouple(8, 1) == (1,)
    assert O.decouple(8, 2) == (1, 5)
    assert O.decouple(8, 4) == (1, 3, 5, 7)
    assert O.decouple(8, 8) == tuple(range(1, 9))
    with pytest.raises(ValueError):
        O.decouple(8, 10)


def test_budgets():
    assert O.budgets_for(0, None) == []
    assert O.budgets_for(1, None) == [2]
    assert O.budgets_for(3, None) == [2, 2, 1]
    assert O.budgets_for(2, 3) == [3, 3]
    with pytest.raises(ValueError):
        O.budgets_for(2, [1])


def test_forward_solve_equals_sequential():
    # SPEC invariant: forward substitution == theta-scheme march
    a, dx = O.laplacian(2, 7, 7)
    d, b = O.blocks_from(a, 0.5, 1e-3)
    u0 = O.bump(2, 7, 7, dx)
    seq = O.sequential(d, b, u0, 16)
    s = O.System(d, b, 16)
    rhs = np.zeros((17, 49))
    rhs[0] = u0
    assert np.abs(O.matvec(s, seq) - rhs).max() < 1e-13


def test_oracle_matches_live_reference(reference):
    from pintmk import solver as R

    from tests.golden.make_golden import reference_hierarchy

    case = SMALL["c3_small"].scaled(name="live", seed=7)
    rh = reference_hierarchy(case)
    xr, rep = R.multilevel_solve(rh)
    oh = oracle_hierarchy(case)
    xo, info = O.solve(oh)
    assert rep.outer_iterations == info["iterations"]
    np.testing.assert_array_equal(xr, xo)
    np.testing.assert_array_equal(np.array(rep.residual_history), np.array(info["history"]))
