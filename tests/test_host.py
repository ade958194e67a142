"""CPU-only checks: C-ABI library exports, host-side setup logic (operators,
stencil tables, sine tables, hierarchy bookkeeping) against the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pintmk_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "pintmk_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(pmk_[a-z0-9_]+)\s*\(",
                                 text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2401_00228_b200 import _lib

    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, n
    assert set(_lib.SIGNATURES) == set(names)
    assert lib.pmk_version().startswith(b"pintmk_b200")


def test_library_is_sm100a():
    from paper_2401_00228_b200 import _lib

    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_ctypes_struct_layout():
    from paper_2401_00228_b200 import _lib

    assert ctypes.sizeof(_lib.Stencil) == 4 + 4 + 40 + 8
    assert ctypes.sizeof(_lib.LevelDesc) == 16 + 2 * 56 + 8


@pytest.mark.parametrize("dim,nx", [(1, 9), (2, 5), (2, 8)])
def test_laplacian_identical_to_oracle(dim, nx):
    import paper_2401_00228_b200 as P

    op = P.build_laplacian(dim, nx, nx if dim == 2 else 1)
    a, dx = O.laplacian(dim, nx, nx if dim == 2 else 1)
    assert op.delta_x == dx
    d = (op.matrix - a)
    assert d.nnz == 0 or np.abs(d.data).max() == 0.0
    assert np.array_equal(op.matrix.indptr, a.indptr)
    assert np.array_equal(op.matrix.indices, a.indices)
    assert np.array_equal(op.matrix.data, a.data)
    np.testing.assert_array_equal(P.initial_bump(op), O.bump(dim, nx, nx if dim == 2 else 1, dx))


def test_stencil_table_constant_and_variable():
    from paper_2401_00228_b200._device import StencilTable

    a, _ = O.laplacian(2, 6, 5)
    d, b = O.blocks_from(a, 0.5, 0.01)
    t = StencilTable(d.T, 6, 5)
    assert t.constant
    assert t.consts[2] == d[0, 0] and t.consts[1] == d[1, 0] and t.consts[0] == d[6, 0]
    groups, (mx, my) = O.agglomerate(7, 7)
    p = O.make_ts_pair(1, 1, groups, 49)
    a7, _ = O.laplacian(2, 7, 7)
    ac = (p.y.T @ a7 @ p.z).tocsr()
    tv = StencilTable(ac.T, mx, my)
    assert not tv.constant
    # reconstruct the matrix from the table
    m = mx * my
    rec = np.zeros((m, m))
    offs = [-mx, -1, 0, 1, mx]
    for s in range(5):
        for i in range(m):
            if tv.coef[s, i] != 0:
                rec[i, i + offs[s]] = tv.coef[s, i]
    np.testing.assert_array_equal(rec, ac.T.toarray())


def test_stencil_table_rejects_wide_pattern():
    from paper_2401_00228_b200._device import StencilTable

    m = sp.csr_matrix(np.ones((9, 9)))
    with pytest.raises(NotImplementedError):
        StencilTable(m, 3, 3)


@pytest.mark.parametrize("nx,ny", [(7, 7), (15, 7), (31, 1)])
def test_sine_tables_diagonalise(nx, ny):
    from paper_2401_00228_b200.spatial import dst_eigenvalues_1d, dst_matrix

    dim = 1 if ny == 1 else 2
    a, dx = O.laplacian(dim, nx, ny)
    sx = dst_matrix(nx)
    np.testing.assert_allclose(sx @ sx, np.eye(nx), atol=1e-13)
    s = sx if ny == 1 else np.kron(dst_matrix(ny), sx)
    lam = (dst_eigenvalues_1d(nx)[None, :] if ny == 1
           else dst_eigenvalues_1d(ny)[:, None] + dst_eigenvalues_1d(nx)[None, :]).ravel()
    lam = lam / dx**2
    np.testing.assert_allclose(s @ a.toarray() @ s, np.diag(lam), atol=1e-9 * abs(lam).max())


def test_agglomerate_partition_matches_oracle():
    from paper_2401_00228_b200 import agglomerate_partition

    for nx, ny in [(7, 1), (8, 1), (7, 7), (6, 9)]:
        g1, s1 = agglomerate_partition(nx, ny)
        g2, s2 = O.agglomerate(nx, ny)
        assert s1 == s2
        assert all(np.array_equal(a, b) for a, b in zip(g1, g2))


@pytest.mark.parametrize("dim,nx,theta,dt,moves", [
    (2, 255, 0.5, 1.6e-7 / 3, 4), (2, 63, 1.0, 2e-3, 2), (2, 15, 0.5, 1e-3, 3),
    (1, 1023, 0.5, 3.05e-7, 3), (1, 63, 1.0, 7.8e-5, 1), (2, 127, 0.3, 1e-5, 3)])
def test_closed_form_stencils_bitwise(dim, nx, theta, dt, moves):
    """The closed-form stencils of pristine levels (SpectralInfo.stencils, used
    instead of scanning the scipy blocks) equal the entries of the blocks the
    reference's formulas produce, bit for bit, on the fine level and on every
    time-coarsened level (a' = 1 - (1 - a)/nu, dt' = nu dt)."""
    from paper_2401_00228_b200 import (ThetaSchemeConfig, build_laplacian,
                                       build_step_operators)
    from paper_2401_00228_b200._device import SpectralInfo, StencilTable
    from paper_2401_00228_b200.solver import _coarse_system_from

    op = build_laplacian(dim, nx, nx if dim == 2 else 1)
    ops = build_step_operators(op, ThetaSchemeConfig(theta, dt, 64))
    factor = op.tau / op.delta_x**2
    ny = op.n_y
    spec = SpectralInfo(factor, theta * dt, (1.0 - theta) * dt)
    def same(mat, want):
        # per-point coefficients (theta = 1 makes phi = I: scipy drops the
        # zero neighbours, the closed form keeps them as 0.0 -- same products)
        got = StencilTable(sp.csr_matrix(mat).T, nx, ny)
        ref = StencilTable.from_constants(want, nx, ny)
        assert np.array_equal(got.coef, ref.coef)
        if got.constant:
            assert np.array_equal(got.consts, want)

    for mat, want in zip((ops.psi, ops.phi), spec.stencils(dim)):
        same(mat, want)
    a, h = theta, dt
    for _ in range(moves):
        a, h = 1.0 - (1.0 - a) / 2, 2 * h
        cs = _coarse_system_from(op.matrix, a, h, 8, (nx, ny), dim, factor)
        assert cs._diag is None  # not assembled by construction
        for mat, want in zip((cs.diag, cs.sub), cs.spectral.stencils(dim)):
            same(mat, want)


@pytest.mark.parametrize("dim,nx,ny,tau,L,theta,dt", [
    (2, 255, 255, 1.0, 1.0, 0.5, 1.6e-7), (2, 63, 17, 0.7, 2.0, 1.0, 1e-3),
    (1, 1023, 1, 1.0, 1.0, 0.5, 3e-7), (1, 17, 1, 2.5, 1.0, 0.0, 1e-2), (2, 1, 1, 1.0, 1.0, 0.5, .1),
    (2, 4, 6, 1.0, 1.0, 0.25, 2e-3), (2, 15, 9, 0.7, 2.0, 1.0, 1e-3), (1, 7, 1, 1.0, 1.0, 1.0, .1)])
def test_direct_csr_assembly_bitwise(dim, nx, ny, tau, L, theta, dt):
    """build_laplacian / build_step_operators assemble the CSR arrays directly;
    they equal (indptr, indices, data, dtypes) scipy's kron / identity /
    scalar-product assembly of the reference's formulas (spatial.py:37-72,
    stepper.py:56-63), including the zero entries scipy drops (theta = 1
    gives phi = I, theta = 0 psi = I)."""
    from paper_2401_00228_b200 import (ThetaSchemeConfig, build_laplacian,
                                       build_step_operators)

    op = build_laplacian(dim, nx, ny, tau=tau, domain_length=L)
    h = L / (nx + 1)
    factor = tau / h**2
    d2 = sp.diags([np.ones(nx - 1), np.full(nx, -2.0), np.ones(nx - 1)], [-1, 0, 1],
                  format="csr")
    if dim == 1:
        ref = (factor * d2).tocsr()
    else:
        dy = sp.diags([np.ones(ny - 1), np.full(ny, -2.0), np.ones(ny - 1)], [-1, 0, 1],
                      format="csr")
        ref = (factor * (sp.kron(sp.identity(ny), d2) + sp.kron(dy, sp.identity(nx)))).tocsr()

    def same(a, b):
        assert a.shape == b.shape and a.indices.dtype == b.indices.dtype
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.data, b.data)

    same(op.matrix, ref)
    ops = build_step_operators(op, ThetaSchemeConfig(theta, dt, 8))
    eye = sp.identity(op.n, format="csr")
    same(ops.phi, (eye + (1.0 - theta) * dt * ref).tocsr())
    same(ops.psi, (eye - theta * dt * ref).tocsr())


def test_hierarchy_bookkeeping_host_only():
    """Level moves / weights / budgets without touching the device."""
    from paper_2401_00228_b200 import solver as S

    assert S.SolverConfig().restart is None
    with pytest.raises(ValueError):
        S.SolverConfig(mu=0.0)
    with pytest.raises(ValueError):
        S.SolverConfig(restart=0)
    levels = [type("L", (), {"budget": 0})() for _ in range(5)]
    S._assign_budgets(levels, None)
    assert [lv.budget for lv in levels] == [0, 2, 2, 1, 0]


def test_product_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_2401_00228_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), fn
            assert "pintmk_oracle" not in src, fn


def test_product_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2401_00228_b200 as P

    op = P.build_laplacian(1, 7)
    ops = P.build_step_operators(op, P.ThetaSchemeConfig(1.0, 0.01, 4))
    with pytest.raises(RuntimeError):
        P.FineSystem(ops, np.zeros(7))
