"""GPU parity of the PCR (1-D parallel cyclic reduction) and LINE (2-D block
Thomas) coarsest solves (csrc/pmk_lines.cu) against the golden fixtures of
the live reference: the kinds are forced with PMK_COARSE_KIND on every small
case they apply to, so they are held to the same bars as the default kinds
(forward_solve <= 1e-12, apply_preconditioner <= 1e-10, full solve +-1
iteration and x <= 1e-10); the mid-size cases where they are the DEFAULT
choice (tests/cases.py line_mid, line_dec_mid, pcr_dec_mid) run in
tests/test_gpu_mid.py."""

import os

import numpy as np
import pytest

from tests.cases import SMALL, gpu_hierarchy

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

ONE_D = sorted(n for n, c in SMALL.items() if c.dim == 1 and c.two_level_family != "MGRIT")
TWO_D = sorted(n for n, c in SMALL.items() if c.dim == 2 and c.two_level_family != "MGRIT")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check(name, kind, monkeypatch):
    from paper_2401_00228_b200 import apply_preconditioner, multilevel_solve

    monkeypatch.setenv("PMK_COARSE_KIND", kind)
    g = golden(name)
    h = gpu_hierarchy(SMALL[name])
    coarse = h.levels[-1].system
    assert coarse.diag_factorization.kind == kind
    out = coarse.forward_solve(g["cs_in"])
    assert rel(out, g["cs_out"]) <= 1e-12, rel(out, g["cs_out"])
    out = apply_preconditioner(h, 0, g["pc_in"])
    assert rel(out, g["pc_out"]) <= 1e-10
    x, rep = multilevel_solve(h)
    assert abs(rep.outer_iterations - int(g["iters"])) <= 1
    assert rel(x, g["x"]) <= 1e-10, rel(x, g["x"])


@pytest.mark.parametrize("name", ONE_D)
def test_pcr_on_every_1d_case(name, monkeypatch):
    _check(name, "pcr", monkeypatch)


@pytest.mark.parametrize("name", TWO_D)
def test_line_on_every_2d_case(name, monkeypatch):
    _check(name, "line", monkeypatch)


def test_pcr_wide_rows_and_many_chains(monkeypatch):
    """m = 2500 (three elements per thread) and 40 chains of unequal length
    against a host Thomas solve of the same chains."""
    import scipy.sparse as sp
    import torch

    from paper_2401_00228_b200._device import CoarseSolver

    rng = np.random.default_rng(7)
    m, n_steps = 2500, 90
    lower, upper = -rng.random(m), -rng.random(m)
    diag = 2.5 + rng.random(m)
    d = sp.diags([lower[1:], diag, upper[:-1]], [-1, 0, 1], format="csr")
    b = sp.diags([0.3 * rng.random(m - 1), 0.5 + rng.random(m), 0.2 * rng.random(m - 1)],
                 [-1, 0, 1], format="csr")
    dropped = tuple(sorted(rng.choice(np.arange(2, n_steps + 1), size=39, replace=False)))
    monkeypatch.setenv("PMK_COARSE_KIND", "pcr")
    cs = CoarseSolver(d, b, n_steps, dropped, 1, m, 1, None)
    assert cs.kind == "pcr"
    rhs = rng.standard_normal((n_steps + 1, m))
    out = torch.empty(rhs.size, dtype=torch.float64, device="cuda")
    cs.solve_into(torch.from_numpy(rhs.ravel()).cuda(), out)
    out = out.cpu().numpy().reshape(n_steps + 1, m)
    dd = d.toarray()
    ref = np.empty_like(rhs)
    ref[0] = rhs[0]
    for k in range(1, n_steps + 1):
        r = rhs[k] if k in dropped else rhs[k] + b @ ref[k - 1]
        ref[k] = np.linalg.solve(dd, r)
    assert rel(out, ref) <= 1e-12, rel(out, ref)


@pytest.mark.parametrize("nx,ny,n_steps,n_cuts", [(100, 37, 6, 0), (300, 9, 5, 2), (40, 50, 40, 30),
                                                   (255, 12, 4, 0), (17, 130, 7, 3)])
def test_line_shapes_against_sparse_lu(nx, ny, n_steps, n_cuts, monkeypatch):
    """Non-square grids, rows per CTA that do not divide nx, lines longer
    than the register-resident variants (streamed G), and cluster sizes 8 / 4
    / 2 / 1 (by chain count), against scipy's sparse LU of the same chains
    (the reference's own coarsest solve, stepper.py:114-146)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    import torch

    from paper_2401_00228_b200._device import CoarseSolver, StencilTable

    rng = np.random.default_rng(nx * 1000 + ny)
    m = nx * ny
    pat = StencilTable._full_pattern(nx, ny)
    indptr, indices, slots = pat[0], pat[1], pat[2]

    def five_point(center, off):
        data = np.where(slots == 2, center + rng.random(slots.size), -off * rng.random(slots.size))
        return sp.csr_matrix((data, indices.copy(), indptr.copy()), shape=(m, m))

    d = five_point(4.5, 1.0)              # strictly diagonally dominant, non-symmetric
    b = five_point(0.5, 0.2)
    dropped = tuple(sorted(int(c) for c in rng.choice(np.arange(2, n_steps + 1), size=n_cuts,
                                                      replace=False))) if n_cuts else ()
    monkeypatch.setenv("PMK_COARSE_KIND", "line")
    cs = CoarseSolver(d, b, n_steps, dropped, 2, nx, ny, None)
    assert cs.kind == "line"
    rhs = rng.standard_normal((n_steps + 1, m))
    out = torch.empty(rhs.size, dtype=torch.float64, device="cuda")
    cs.solve_into(torch.from_numpy(rhs.ravel()).cuda(), out)
    out = out.cpu().numpy().reshape(n_steps + 1, m)
    lu = spla.splu(sp.csc_matrix(d))
    bt = sp.csr_matrix(b.T)               # 2-D couples with B^T (stepper.py:144)
    ref = np.empty_like(rhs)
    ref[0] = rhs[0]
    for k in range(1, n_steps + 1):
        r = rhs[k] if k in dropped else rhs[k] + bt @ ref[k - 1]
        ref[k] = lu.solve(r)
    assert rel(out, ref) <= 1e-12, rel(out, ref)
