"""The small host-side helpers the package mirrors from the reference's
intergrid.py (closed_form_t_coarse, build_t_pair, build_ts_pair,
build_mgrit_pair, block_matrices, materialize) against the LIVE reference
(CPU; skipped where /root/reference is absent, e.g. on the GPU box)."""

import types

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2401_00228_b200 as P
from paper_2401_00228_b200 import intergrid as G


def _same(a, b):
    a, b = sp.csr_matrix(a), sp.csr_matrix(b)
    assert a.shape == b.shape
    assert abs(a - b).max() == 0.0 if a.nnz or b.nnz else True


@pytest.mark.parametrize("dim,n,nu,n_T", [(1, 15, 2, 8), (2, 7, 3, 4)])
def test_time_pair_helpers_match_reference(reference, dim, n, nu, n_T):
    from pintmk import intergrid as R

    m = n * (n if dim == 2 else 1)
    ours, ref = G.build_t_pair(m, nu, n_T), R.build_t_pair(m, nu, n_T)
    assert (ours.n, ours.nu, ours.n_T, ours.fine_rows) == (ref.n, ref.nu, ref.n_T, ref.fine_rows)
    for k in (0, 1, n_T):
        for a, b in zip(ours.block_matrices(k), ref.block_matrices(k)):
            _same(a, b)
    for a, b in zip(ours.materialize(), ref.materialize()):
        _same(a, b)


@pytest.mark.parametrize("nx,ny,nu", [(15, 1, 2), (7, 7, 2), (15, 15, 1)])
def test_time_space_pair_helpers_match_reference(reference, nx, ny, nu):
    from pintmk import intergrid as R

    groups, _ = G.agglomerate_partition(nx, ny)
    rgroups, _ = R.agglomerate_partition(nx, ny)
    for a, b in zip(groups, rgroups):
        np.testing.assert_array_equal(np.sort(a), np.sort(b))
    ours = G.build_ts_pair(nx * ny, nu, 4, groups)
    ref = R.build_ts_pair(nx * ny, nu, 4, rgroups)
    _same(ours.y_space, ref.y_space)
    _same(ours.z_space, ref.z_space)
    for k in (0, 1):
        for a, b in zip(ours.block_matrices(k), ref.block_matrices(k)):
            _same(a, b)
    for a, b in zip(ours.materialize(), ref.materialize()):
        _same(a, b)


@pytest.mark.parametrize("dim,theta,nu", [(1, 0.5, 2), (2, 1.0, 4)])
def test_closed_form_t_coarse_matches_reference(reference, dim, theta, nu):
    from pintmk import spatial as RS
    from pintmk import stepper as RT
    from pintmk import intergrid as R

    n = 15 if dim == 1 else 7
    dt = 1e-3
    ops = P.build_step_operators(P.build_laplacian(dim, n, n if dim == 2 else 1),
                                 P.ThetaSchemeConfig(theta, dt, 8))
    rops = RT.build_step_operators(RS.build_laplacian(dim, n, n if dim == 2 else 1),
                                   RT.ThetaSchemeConfig(theta, dt, 8))
    ours = G.closed_form_t_coarse(ops, nu, 8 // nu)
    ref = R.closed_form_t_coarse(rops, nu, 8 // nu)
    _same(ours.diag, ref.diag)
    _same(ours.sub, ref.sub)
    assert ours.n_steps == ref.n_steps and ours.provenance == ref.provenance


def test_build_mgrit_pair_reads_the_partition():
    ops = P.build_step_operators(P.build_laplacian(1, 15), P.ThetaSchemeConfig(0.5, 1e-3, 8))
    part = types.SimpleNamespace(fine=types.SimpleNamespace(ops=ops), nu=2, n_T=4)
    pair = G.build_mgrit_pair(part)
    assert (pair.nu, pair.n_T, pair.fine_rows, pair.n) == (2, 4, 9, 15)
