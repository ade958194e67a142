"""Host logic of the PCR and LINE coarsest solves (CPU only): the tables
built by _device.pcr_tables / line_tables, run through a numpy restatement of
exactly what csrc/pmk_lines.cu does per slice (cyclic-reduction sweeps of the
right-hand side; block Thomas over grid lines), reproduce the oracle's
forward_solve (the reference's Thomas chain / SuperLU per slice,
stepper.py:114-146) to rounding, for exact and decoupled chains."""

import numpy as np
import pytest

from oracle import pintmk_oracle as O
from paper_2401_00228_b200._device import StencilTable, line_tables, pcr_tables
from tests.cases import SMALL, Case, oracle_hierarchy


def chain_rows(n_steps, dropped):
    cuts = sorted(c for c in dropped if c > 1)
    return list(zip([1] + cuts, cuts + [n_steps + 1]))


def coupling_apply(coef, nx, ny, prev):
    """Row-form 5-slot stencil times a slice (the kernels' coupling step)."""
    m = nx * ny
    out = coef[2] * prev
    out[1:] += (coef[1] * np.concatenate([[0.0], prev[:-1]]))[1:]
    out[:-1] += (coef[3] * np.concatenate([prev[1:], [0.0]]))[:-1]
    if ny > 1:
        out[nx:] += coef[0][nx:] * prev[:m - nx]
        out[:m - nx] += coef[4][:m - nx] * prev[nx:]
    return out


def emulate_pcr(system, m, rhs):
    d = StencilTable(system.diag, m, 1).coef
    c = StencilTable(system.sub, m, 1).coef          # 1-D couples with B itself
    alpha, gamma, inv = pcr_tables(d[1], d[2], d[3])
    r = rhs.reshape(system.n_steps + 1, m)
    out = np.empty_like(r)
    out[0] = r[0]
    for first, end in chain_rows(system.n_steps, system.dropped):
        cut = first in system.dropped
        x = np.zeros(m) if cut else r[first - 1].copy()
        for k in range(first, end):
            v = r[k].copy() if (k == first and cut) else r[k] + coupling_apply(c, m, 1, x)
            for lv in range(alpha.shape[0]):
                s = 1 << lv
                nv = v.copy()
                nv[s:] += alpha[lv, s:] * v[:-s]
                nv[:-s] += gamma[lv, :-s] * v[s:]
                v = nv
            x = v * inv
            out[k] = x
    return out.reshape(-1)


def emulate_line(system, nx, ny, rhs):
    m = nx * ny
    d = StencilTable(system.diag, nx, ny).coef
    c = StencilTable(system.sub.T, nx, ny).coef      # 2-D couples with B^T
    g = line_tables(d, nx, ny)
    lo, up = d[0].reshape(ny, nx), d[4].reshape(ny, nx)
    r = rhs.reshape(system.n_steps + 1, m)
    out = np.empty_like(r)
    out[0] = r[0]
    for first, end in chain_rows(system.n_steps, system.dropped):
        cut = first in system.dropped
        for k in range(first, end):
            b = r[k].copy() if (k == first and cut) else r[k] + coupling_apply(c, nx, ny, out[k - 1])
            b = b.reshape(ny, nx)
            y = np.empty((ny, nx))
            for j in range(ny):
                t = b[j] - lo[j] * y[j - 1] if j > 0 else b[j]
                y[j] = g[j] @ t
            x = np.empty((ny, nx))
            x[ny - 1] = y[ny - 1]
            for j in range(ny - 2, -1, -1):
                x[j] = y[j] - g[j] @ (up[j] * x[j + 1])
            out[k] = x.reshape(-1)
    return out.reshape(-1)


PCR_CASES = [SMALL[n] for n in ("c1_small", "c1_lit_small", "c2_small", "ts2_small",
                                "long1_dec_small", "np2_1d_small", "rowscale_1d_small",
                                "forced_1d_small")] + [
    Case("agg1_host", 1, 63, 32, 0.5, 3, ("time", "space"), courant=0.64, n_cgs=5),
    Case("one_point", 1, 1, 8, 1.0, 2, ("time",), courant=0.64),
    Case("wide_1d", 1, 1500, 4, 0.5, 2, ("time",), courant=0.64, perturb="rowscale"),
]

LINE_CASES = [SMALL[n] for n in ("c3_small", "c5_small", "space_small", "rowscale_small",
                                 "rowscale_dec_small", "np2_2d_small", "even_space_small")]


@pytest.mark.parametrize("case", PCR_CASES, ids=lambda c: c.name)
def test_pcr_restatement_matches_reference_forward_solve(case):
    s = oracle_hierarchy(case).rungs[-1].system
    rhs = np.random.default_rng(1).standard_normal(s.size)
    ref = O.forward_solve(s, rhs)
    out = emulate_pcr(s, s.n, rhs)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-13


@pytest.mark.parametrize("case", LINE_CASES, ids=lambda c: c.name)
def test_line_restatement_matches_reference_forward_solve(case):
    rung = oracle_hierarchy(case).rungs[-1]
    s = rung.system
    rhs = np.random.default_rng(2).standard_normal(s.size)
    ref = O.forward_solve(s, rhs)
    out = emulate_line(s, rung.grid[0], rung.grid[1], rhs)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) <= 1e-13


def test_pcr_tables_reduce_to_a_diagonal_system():
    rng = np.random.default_rng(3)
    m = 37
    lower, upper = -rng.random(m), -rng.random(m)
    diag = 2.5 + rng.random(m)
    alpha, gamma, inv = pcr_tables(lower, diag, upper)
    assert alpha.shape == (6, m)
    a = np.diag(diag) + np.diag(lower[1:], -1) + np.diag(upper[:-1], 1)
    for lv in range(alpha.shape[0]):
        s = 1 << lv
        e = np.eye(m)
        e[np.arange(s, m), np.arange(m - s)] = alpha[lv, s:]
        e[np.arange(m - s), np.arange(s, m)] = gamma[lv, :-s]
        a = e @ a
    off = a - np.diag(np.diag(a))
    assert np.abs(off).max() <= 1e-14
    assert np.allclose(np.diag(a) * inv, 1.0, rtol=1e-14)


def test_zero_pivot_raises_like_the_reference():
    with pytest.raises(np.linalg.LinAlgError, match="factorization failed"):
        pcr_tables(np.zeros(4), np.array([1.0, 0.0, 1.0, 1.0]), np.zeros(4))


def test_line_chunks_layout_and_cluster_size():
    from paper_2401_00228_b200._device import line_chunks, line_cluster_size

    g = np.random.default_rng(5).standard_normal((3, 13, 13))
    for cs in (1, 2, 4, 8):
        ch = line_chunks(g, cs)
        r = -(-13 // cs)
        assert ch.shape == (3, cs, r, 13)
        for q in range(cs):
            for rr in range(r):
                row = q * r + rr
                want = g[:, row, :] if row < 13 else np.zeros((3, 13))
                np.testing.assert_array_equal(ch[:, q, rr, :], want)
    assert [line_cluster_size(n) for n in (1, 18, 19, 37, 74, 75, 500)] == [8, 8, 4, 4, 2, 1, 1]
