"""GPU parity of the full-weighting / bilinear space moves (EXTENSION, see
tests/test_fw_host.py: no reference counterpart; the checker is the oracle's
restatement of the same formulas, and everything around the transfers is the
reference-pinned path).  Bars as for the reference-backed cases: transfers
<= 1e-14 relative (same products, fixed order), level operators equal,
apply_preconditioner <= 1e-10, solve iteration count +-1 and x <= 1e-10."""

import numpy as np
import pytest

from tests.cases import FW, gpu_hierarchy, oracle_hierarchy

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", sorted(FW))
def test_fw_moves_against_the_oracle(name):
    from oracle import pintmk_oracle as O
    from paper_2401_00228_b200 import apply_preconditioner, multilevel_solve

    case = FW[name]
    h = gpu_hierarchy(case)
    oh = oracle_hierarchy(case)
    assert list(h.moves) == oh.moves
    rng = np.random.default_rng(11)
    for lv, r in zip(h.levels, oh.rungs):
        assert lv.grid == r.grid and lv.n_steps == r.n_steps
        v = rng.standard_normal(r.system.size)
        np.testing.assert_array_equal(lv.system.matvec(v), O.matvec(r.system, v))
    for lv, r in zip(h.levels[:-1], oh.rungs[:-1]):
        v = rng.standard_normal(r.system.size)
        got, want = lv.pair.restrict(v), O.restrict(r.pair, v)
        assert rel(got, want) <= 1e-14, rel(got, want)
        w = rng.standard_normal(want.size)
        got, want = lv.pair.interpolate(w), O.interpolate(r.pair, w)
        assert rel(got, want) <= 1e-14, rel(got, want)
    cs = rng.standard_normal(oh.rungs[-1].system.size)
    assert rel(h.levels[-1].system.forward_solve(cs),
               O.forward_solve(oh.rungs[-1].system, cs)) <= 1e-12
    v = rng.standard_normal(oh.rungs[0].system.size)
    assert rel(apply_preconditioner(h, 0, v), O.precondition(oh, 0, v)) <= 1e-10
    x, rep = multilevel_solve(h)
    xo, info = O.solve(oh)
    assert abs(rep.outer_iterations - info["iterations"]) <= 1
    assert rel(x, xo) <= 1e-10, rel(x, xo)
    n = min(len(rep.residual_history), len(info["history"]))
    np.testing.assert_allclose(rep.residual_history[:n], info["history"][:n], rtol=1e-6)


def test_fw_move_needs_a_pristine_laplacian_and_odd_grids():
    import paper_2401_00228_b200 as P
    from tests.cases import SMALL, Case

    with pytest.raises(ValueError, match="build_laplacian"):
        gpu_hierarchy(SMALL["rowscale_small"].scaled(schedule=("space_fw", "time")))
    with pytest.raises(ValueError, match="odd"):
        gpu_hierarchy(Case("even", 2, 12, 16, 0.5, 2, ("space_fw",), courant=0.16))
    assert P.WeightedSpacePair(2, 4, (7, 7), 2).coarse_grid == (3, 3)
