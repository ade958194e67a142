"""Host side of the full-weighting / bilinear space moves (EXTENSION: BASELINE
config 4 names these transfers, the reference only agglomerates, so there is
no reference output to pin to).  CPU only: the product's transfer matrices
and rediscretised coarse operators equal the oracle's restatement bit for
bit, the weights have the textbook properties, and the oracle solve with
these moves converges."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pintmk_oracle as O
from paper_2401_00228_b200.intergrid import full_weighting_1d
from tests.cases import FW, oracle_hierarchy


def test_weights_1d():
    r, p = full_weighting_1d(7)
    assert r.shape == (3, 7) and p.shape == (7, 3)
    np.testing.assert_array_equal(r.toarray()[1], [0, 0, 0.25, 0.5, 0.25, 0, 0])
    np.testing.assert_array_equal(p.toarray()[:, 1], [0, 0, 0.5, 1.0, 0.5, 0, 0])
    assert np.all(np.asarray(r.sum(axis=1)).ravel() == 1.0)
    ro, po = O.fw_1d(7)
    np.testing.assert_array_equal(r.toarray(), ro.toarray())
    np.testing.assert_array_equal(p.toarray(), po.toarray())
    for bad in (1, 2, 8):
        with pytest.raises(ValueError):
            full_weighting_1d(bad)


def test_linear_functions_are_interpolated_exactly():
    """Bilinear interpolation reproduces functions linear in x and y that
    vanish on the boundary corner rows it cannot see: check the interior."""
    nx = 15
    p = O.make_fw_pair(1, 1, nx, nx, 2)
    xc = np.arange(1, 8) / 8.0
    xf = np.arange(1, 16) / 16.0
    wc = np.add.outer(2.0 * xc, 3.0 * xc).ravel()
    wf = np.add.outer(2.0 * xf, 3.0 * xf)
    got = (p.z @ wc).reshape(nx, nx)
    np.testing.assert_allclose(got[1:-1, 1:-1], wf[1:-1, 1:-1], rtol=1e-15)


@pytest.mark.parametrize("name", sorted(FW))
def test_oracle_solve_with_fw_moves_converges(name):
    case = FW[name]
    h = oracle_hierarchy(case)
    assert h.moves == list(case.schedule)
    x, info = O.solve(h)
    if name == "fw_c4_small":  # nu = 4 with space coarsening: slow, like c4_small (agglomeration)
        assert info["iterations"] == case.max_outer and info["history"][-1] < 2e-3
    else:
        assert info["iterations"] < case.max_outer
        assert O.relative_residual(h, x) <= 1e-8
    # coarse grids halve the spacing count: (n - 1) / 2
    for r0, r1, mv in zip(h.rungs[:-1], h.rungs[1:], h.moves):
        if mv.endswith("_fw"):
            assert r1.grid[0] == (r0.grid[0] - 1) // 2
            # rediscretised: a pristine Laplacian with a quarter of the factor
            assert r1.a[0, 1] == r0.a[0, 1] / 4.0
            assert sp.issparse(r0.pair.y) and r0.pair.y.shape == (r0.a.shape[0], r1.a.shape[0])
