"""Host logic of the EIG coarsest solve (CPU only): SeparableFactors detects
D = I - K, B = I + b K with K a Kronecker sum of tridiagonals on the
coarsest systems the reference builds, and a numpy restatement of the device
algorithm (eigen-transforms, per-mode recurrence, the 2-D low-rank B^T
correction of csrc/pmk_coarse.cu eig_chain_kernel) reproduces the oracle's
forward_solve (the reference's LU / Thomas chain) to rounding."""

import numpy as np
import pytest

from oracle import pintmk_oracle as O
from paper_2401_00228_b200._device import SeparableFactors
from tests.cases import SMALL, Case, oracle_hierarchy


def emulate(fac, nx, ny, dim, n_steps, dropped, rhs):
    r = rhs.reshape(n_steps + 1, ny, nx)
    rh = np.einsum("qj,kjp->kqp", fac.vyi, np.einsum("kyx,px->kyp", r, fac.vxi))
    delta, beta = (t.reshape(ny, nx) for t in fac.mode_tables())
    z = np.empty_like(rh)
    z[0] = rh[0]
    for k in range(1, n_steps + 1):
        if k in dropped:
            z[k] = rh[k] / delta
            continue
        prev = z[k - 1]
        corr = np.zeros_like(prev)
        if dim == 2 and fac.corr_x is not None:
            h, u = fac.corr_x
            corr += (prev @ h.T) @ u
        if dim == 2 and fac.corr_y is not None:
            h, u = fac.corr_y
            corr += u.T @ (h @ prev)
        z[k] = (rh[k] + beta * prev + fac.b * corr) / delta
    out = np.einsum("qj,kjp->kqp", fac.vy, np.einsum("kyp,xp->kyx", z, fac.vx))
    out[0] = r[0]
    return out.reshape(-1)


CASES = [SMALL[n] for n in ("c2_small", "c4_small", "space_small", "ts2_small",
                            "auto_small", "even_space_small", "space_dec_small",
                            "rowscale_1d_small")] + [
    Case("ttts_host", 2, 31, 32, 0.5, 5, ("time", "time", "time", "space"), courant=0.16),
    Case("ss_host", 2, 31, 16, 1.0, 3, ("space", "space"), courant=0.16),
    Case("agg1_host", 1, 63, 32, 0.5, 3, ("time", "space"), courant=0.64, n_cgs=5),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c.name)
def test_eig_restatement_matches_reference_forward_solve(case):
    h = oracle_hierarchy(case)
    c = h.rungs[-1]
    s = c.system
    nx, ny = c.grid[0], (c.grid[1] if c.dim == 2 else 1)
    fac = SeparableFactors.detect(s.diag, s.sub, nx, ny, c.dim)
    assert fac is not None
    rhs = np.random.default_rng(0).standard_normal(s.size)
    ref = O.forward_solve(s, rhs)
    out = emulate(fac, nx, ny, c.dim, s.n_steps, set(s.dropped), rhs)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-13


def test_odd_grid_agglomeration_needs_a_rank_two_correction():
    h = oracle_hierarchy(SMALL["space_small"])
    c = h.rungs[-1]
    fac = SeparableFactors.detect(c.system.diag, c.system.sub, *c.grid, c.dim)
    # the 3-wide last group: one asymmetric pair per direction -> 2 points
    assert fac.corr_x[0].shape == (2, c.grid[0]) and fac.corr_y[0].shape == (2, c.grid[1])


def test_non_separable_operator_is_rejected():
    h = oracle_hierarchy(SMALL["rowscale_small"])
    c = h.rungs[-1]
    assert SeparableFactors.detect(c.system.diag, c.system.sub, *c.grid, c.dim) is None
