"""GPU parity: the sm_100a path (through the public API / C-ABI) against the
CPU oracle and the committed golden fixtures of the reference.

Tolerances (fp64):
  * matvec, restrict, interpolate: bitwise (same operations, same order);
  * coarsest forward_solve: <= 1e-12 relative l2 (sine-diagonalised /
    dense-inverse solve vs the reference's LU / Thomas: rounding only);
  * apply_preconditioner (contains inner FGMRES + coarsest solve): <= 1e-10;
  * full solve: same iteration count (+-1) and x within 1e-10 relative l2 of
    the reference (the north-star parity bar).
"""

import os

import numpy as np
import pytest

from tests.cases import SMALL, gpu_hierarchy, oracle_hierarchy

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


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


@pytest.mark.parametrize("name", sorted(SMALL))
def test_matvec_bitwise(name):
    g = golden(name)
    h = gpu_hierarchy(SMALL[name])
    out = h.levels[0].system.matvec(g["mv_in"])
    np.testing.assert_array_equal(out, g["mv_out"])


@pytest.mark.parametrize("name", sorted(SMALL))
def test_transfers_bitwise(name):
    """Restrictions are bitwise; interpolations are bitwise except the MGRIT
    family's ideal interpolation, whose (psi^{-1} phi)^j propagation runs in
    the sine basis (reference: per-step LU/Thomas solves): <= 1e-13."""
    from paper_2401_00228_b200.intergrid import MgritPair

    g = golden(name)
    h = gpu_hierarchy(SMALL[name])
    for i, lv in enumerate(h.levels[:-1]):
        np.testing.assert_array_equal(lv.pair.restrict(g[f"r{i}_in"]), g[f"r{i}_out"])
        out = lv.pair.interpolate(g[f"i{i}_in"])
        if isinstance(lv.pair, MgritPair):
            assert rel(out, g[f"i{i}_out"]) <= 1e-13, rel(out, g[f"i{i}_out"])
        else:
            np.testing.assert_array_equal(out, g[f"i{i}_out"])


@pytest.mark.parametrize("name", sorted(SMALL))
def test_coarsest_forward_solve(name):
    g = golden(name)
    h = gpu_hierarchy(SMALL[name])
    out = h.levels[-1].system.forward_solve(g["cs_in"])
    assert rel(out, g["cs_out"]) <= 1e-12


@pytest.mark.parametrize("name", sorted(SMALL))
def test_apply_preconditioner(name):
    from paper_2401_00228_b200 import apply_preconditioner

    g = golden(name)
    h = gpu_hierarchy(SMALL[name])
    out = apply_preconditioner(h, 0, g["pc_in"])
    assert rel(out, g["pc_out"]) <= 1e-10


@pytest.mark.parametrize("name", sorted(SMALL))
def test_solve_parity(name):
    from paper_2401_00228_b200 import multilevel_solve

    case = SMALL[name]
    g = golden(name)
    h = gpu_hierarchy(case)
    x, rep = multilevel_solve(h)
    assert abs(rep.outer_iterations - int(g["iters"])) <= 1
    assert rel(x, g["x"]) <= 1e-10, rel(x, g["x"])
    hist = np.array(rep.residual_history)
    k = min(len(hist), len(g["hist"]))
    assert np.allclose(hist[:k], g["hist"][:k], rtol=1e-6, atol=1e-14)


@pytest.mark.parametrize("name", ["c3_small", "c5_small"])
def test_fgmres_internals_vs_oracle(name):
    """Basis, preconditioned vectors and Hessenberg of a 3-iteration solve."""
    from oracle import pintmk_oracle as O
    from paper_2401_00228_b200 import fgmres

    case = SMALL[name]
    h = gpu_hierarchy(case)
    oh = oracle_hierarchy(case)
    rhs = oh.rhs.ravel()
    x, rep = fgmres(h, 0, rhs, tol=None, max_iter=3, keep_basis=True)
    xo, info = O.fgmres(oh, 0, rhs, None, 3, keep_basis=True)
    assert rep.outer_iterations == info["iterations"] == 3
    for a, b in zip(rep.metadata["basis"], info["basis"]):
        assert rel(a, b) <= 1e-11
    for a, b in zip(rep.metadata["preconditioned"], info["preconditioned"]):
        assert rel(a, b) <= 1e-11
    np.testing.assert_allclose(rep.metadata["hessenberg"], info["hessenberg"], rtol=1e-10,
                               atol=1e-13)
    assert rel(x, xo) <= 1e-10


@pytest.mark.parametrize("name", ["c3_small", "c5_small", "c2_small"])
def test_orthogonality_and_arnoldi_relation(name):
    """SURVEY section 4 known answers: the one-reduce orthogonalisation loses
    orthogonality like the reference's MGS (c3_small: 9.6e-8 both after 12
    iterations) and the Arnoldi relation A Z = V H holds to rounding."""
    from oracle import pintmk_oracle as O
    from paper_2401_00228_b200 import fgmres

    case = SMALL[name]
    h = gpu_hierarchy(case)
    oh = oracle_hierarchy(case)
    rhs = oh.rhs.ravel()
    _, rep = fgmres(h, 0, rhs, tol=None, max_iter=12, keep_basis=True)
    _, info = O.fgmres(oh, 0, rhs, None, 12, keep_basis=True)

    def loss(basis):
        V = np.stack(basis, axis=1)
        return float(np.abs(V.T @ V - np.eye(V.shape[1])).max())

    ours, ref = loss(rep.metadata["basis"]), loss(info["basis"])
    assert ours <= 4.0 * ref + 1e-13, (ours, ref)
    Z = np.stack(rep.metadata["preconditioned"], axis=1)
    V = np.stack(rep.metadata["basis"][:Z.shape[1] + 1], axis=1)
    AZ = np.stack([O.matvec(oh.fine, Z[:, j]) for j in range(Z.shape[1])], axis=1)
    arn = np.linalg.norm(AZ - V @ rep.metadata["hessenberg"]) / np.linalg.norm(AZ)
    assert arn <= 1e-14, arn


_CLASSIC_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from tests.cases import SMALL, gpu_hierarchy, oracle_hierarchy
from oracle import pintmk_oracle as O
from paper_2401_00228_b200 import fgmres, multilevel_solve
out = {}
for name in ("c5_small", "mgrit2_small"):
    case = SMALL[name]
    h = gpu_hierarchy(case)
    oh = oracle_hierarchy(case)
    rhs = oh.rhs.ravel()
    x, rep = fgmres(h, 0, rhs, tol=None, max_iter=3, keep_basis=True)
    xo, info = O.fgmres(oh, 0, rhs, None, 3, keep_basis=True)
    hd = np.abs(rep.metadata["hessenberg"] - info["hessenberg"]).max()
    g = np.load(f"{sys.argv[1]}/tests/golden/{name}.npz")
    xs, rs = multilevel_solve(gpu_hierarchy(case))
    out[name] = {"hdiff": float(hd), "iters": rs.outer_iterations, "g_iters": int(g["iters"]),
                 "xrel": float(np.linalg.norm(xs - g["x"]) / np.linalg.norm(g["x"]))}
print(json.dumps(out))
"""


def test_classic_mgs_mode():
    """PMK_MGS=classic (one basis vector per pass in the reference's order,
    exact division for the normalised basis vectors) meets the same parity
    bar as the default one-reduce orthogonalisation."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PMK_MGS="classic")
    r = subprocess.run([sys.executable, "-c", _CLASSIC_SCRIPT, root], env=env, cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, d in res.items():
        assert d["hdiff"] <= 1e-12, (name, d)
        assert abs(d["iters"] - d["g_iters"]) <= 1, (name, d)
        assert d["xrel"] <= 1e-10, (name, d)


def test_solve_is_deterministic():
    from paper_2401_00228_b200 import multilevel_solve

    case = SMALL["c5_small"]
    x1, r1 = multilevel_solve(gpu_hierarchy(case))
    x2, r2 = multilevel_solve(gpu_hierarchy(case))
    np.testing.assert_array_equal(x1, x2)
    assert r1.residual_history == r2.residual_history


def test_device_io_roundtrip():
    """A device-resident u0 gives a device x equal to the host path's."""
    import torch

    from paper_2401_00228_b200 import multilevel_solve

    case = SMALL["c3_small"]
    xh, _ = multilevel_solve(gpu_hierarchy(case))
    xd, _ = multilevel_solve(gpu_hierarchy(case, u0=torch.from_numpy(case.u0_vector()).cuda()))
    assert isinstance(xd, torch.Tensor) and xd.is_cuda
    np.testing.assert_array_equal(xd.cpu().numpy(), xh)


@pytest.mark.parametrize("name", ["c1_small", "c2_small", "c4_small", "c5_small",
                                  "ts2_small", "mgrit1_small", "mgrit2_dec_small"])
def test_host_output_slabs_bitwise(name):
    """x assembled slab by slab (pmk_fgmres_finish_rows) and streamed into a
    host buffer equals the one-launch device assembly bitwise: time pairs
    (nu = 2, 4), agglomerated TS pairs, MGRIT, with and without restarts."""
    import torch

    from paper_2401_00228_b200 import multilevel_solve

    case = SMALL[name]
    for restart in (None, 5):
        c = case.scaled(restart=restart) if restart else case
        u0 = torch.from_numpy(c.u0_vector())
        xd, rd = multilevel_solve(gpu_hierarchy(c, u0=u0.cuda()))
        pin = torch.full((c.N,), float("nan"), dtype=torch.float64).pin_memory()
        xo, ro = multilevel_solve(gpu_hierarchy(c, u0=u0.cuda()), out=pin)
        assert xo is pin
        np.testing.assert_array_equal(pin.numpy(), xd.cpu().numpy())
        xn, _ = multilevel_solve(gpu_hierarchy(c))  # numpy in -> numpy out
        assert isinstance(xn, np.ndarray)
        np.testing.assert_array_equal(xn, xd.cpu().numpy())
        assert ro.outer_iterations == rd.outer_iterations


@pytest.mark.parametrize("budgets", [(3, 2, 1), (2, 3, 2), (4, 1, 2)])
def test_inner_budgets_vs_oracle(budgets):
    """Fixed inner budgets other than the default [2, 2, 1] (SolverConfig
    inner_iters, solver.py:219-235) against the CPU oracle: exercises the
    deferred first orthogonalisation of fgmres_fixed with budgets > 2 (step 1
    writing into slot 2) and a budget-1 level between fused ones."""
    from oracle import pintmk_oracle as O
    from paper_2401_00228_b200 import multilevel_solve

    case = SMALL["c5_small"].scaled(inner_iters=budgets)
    x, rep = multilevel_solve(gpu_hierarchy(case))
    xo, info = O.solve(oracle_hierarchy(case))
    assert abs(rep.outer_iterations - info["iterations"]) <= 1
    assert rel(x, xo) <= 1e-10, rel(x, xo)


@pytest.mark.parametrize("name", ["c5_small", "c4_small", "mgrit2_small", "c2_small"])
def test_lazy_basis_matches_normalised_basis(name):
    """The lazy Krylov basis (default) against the explicitly normalised one
    (PMK_LAZY=0, run in a subprocess: the mode is fixed per process): same
    iterations, x within 1e-12 (only where the scales are folded -- dot
    products, update coefficients -- does the rounding differ)."""
    import json
    import subprocess
    import sys
    import tempfile

    from paper_2401_00228_b200 import _lib, multilevel_solve

    assert _lib.lazy_basis()
    case = SMALL[name]
    x, rep = multilevel_solve(gpu_hierarchy(case))
    code = ("import json,sys; sys.path.insert(0, %r); import numpy as np; "
            "from tests.cases import SMALL, gpu_hierarchy; "
            "from paper_2401_00228_b200 import _lib, multilevel_solve; "
            "assert not _lib.lazy_basis(); "
            "x, r = multilevel_solve(gpu_hierarchy(SMALL[%r])); "
            "np.save(sys.argv[1], x); print(json.dumps(r.outer_iterations))"
            % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), name))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.npy")
        env = dict(os.environ, PMK_LAZY="0")
        out = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True,
                             text=True, check=True)
        xn = np.load(path)
    assert json.loads(out.stdout.strip().splitlines()[-1]) == rep.outer_iterations
    assert rel(x, xn) <= 1e-12, rel(x, xn)


def test_sequential_solve_matches_oracle():
    from oracle import pintmk_oracle as O
    from paper_2401_00228_b200 import (ThetaSchemeConfig, build_laplacian,
                                       build_step_operators, sequential_solve)

    case = SMALL["c3_small"]
    op = build_laplacian(2, case.nx, case.nx)
    ops = build_step_operators(op, ThetaSchemeConfig(case.theta, case.dt(), case.n_t))
    u0 = case.u0_vector()
    out = sequential_solve(ops, u0)
    a, _ = O.laplacian(2, case.nx, case.nx)
    d, b = O.blocks_from(a, case.theta, case.dt())
    ref = O.sequential(d, b, u0, case.n_t)
    assert rel(out, ref) <= 1e-12


def test_zero_rhs_returns_zero():
    from paper_2401_00228_b200 import fgmres

    h = gpu_hierarchy(SMALL["c3_small"])
    x, rep = fgmres(h, 0, np.zeros(h.levels[0].total_dim), tol=1e-8, max_iter=5)
    assert float(abs(x).max()) == 0.0 and rep.outer_iterations == 0


def test_bad_shapes_raise():
    import paper_2401_00228_b200 as P

    h = gpu_hierarchy(SMALL["c3_small"])
    with pytest.raises(ValueError):
        h.levels[0].system.matvec(np.zeros(7))
    with pytest.raises(ValueError):
        P.apply_preconditioner(h, 2, np.zeros(h.levels[2].total_dim))


@pytest.mark.parametrize("dim,nx,ny,n_t,theta", [(1, 1023, 1, 16, 0.5), (2, 300, 20, 8, 0.5),
                                                 (2, 255, 9, 6, 1.0), (1, 255, 1, 12, 0.5),
                                                 (2, 256, 5, 4, 0.5), (1, 17, 1, 9, 0.3),
                                                 (1, 700, 1, 10, 1.0), (2, 509, 7, 4, 0.5)])
def test_fused_kernels_bitwise_wide_and_odd_grids(dim, nx, ny, n_t, theta):
    """K-MV, K-MVR (shift + restrict + normalised copy) and K-IMV against the
    oracle's operations, on grids wider than one 255-column tile and with odd
    row lengths (TMA parity shifts)."""
    import ctypes

    import torch

    from oracle import pintmk_oracle as O
    from paper_2401_00228_b200 import _lib
    from paper_2401_00228_b200.intergrid import TimePair
    from paper_2401_00228_b200.stepper import BlockBidiagonalSystem

    a, _ = O.laplacian(dim, nx, ny)
    d, b = O.blocks_from(a, theta, 1e-4)
    nu = 2 if n_t % 2 == 0 else 3 if n_t % 3 == 0 else 1
    sysd = BlockBidiagonalSystem(d, b, n_t, grid=(nx, ny), dim=dim)
    so = O.System(d, b, n_t)
    pair = TimePair(nx * ny, nu, n_t // nu)
    po = O.Pair(nu, n_t // nu, nx * ny)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(so.size)
    scale = 3.7
    # K-MV
    np.testing.assert_array_equal(sysd.matvec(v), O.matvec(so, v))
    # K-MVR with lazy scale: vh = restrict(A v - mu v), v_norm = raw / scale
    lib = _lib.load()
    raw = torch.from_numpy(v * scale).cuda()
    sc = torch.tensor([scale], dtype=torch.float64, device="cuda")
    vh = torch.empty((n_t // nu + 1) * nx * ny, dtype=torch.float64, device="cuda")
    _lib.check(lib.pmk_stmv_shift_restrict(ctypes.byref(sysd.level_desc()),
                                           ctypes.byref(pair._pair_desc()), 0.75, _lib.ptr(raw),
                                           _lib.ptr(sc), _lib.ptr(vh), None, _lib.stream_ptr()),
               "mvr")
    vn = (v * scale) / scale
    s_ref = O.matvec(so, vn)
    s_ref -= 0.75 * vn
    np.testing.assert_array_equal(vh.cpu().numpy(), O.restrict(po, s_ref))
    # K-IMV: x = v - Z vt, w = A x
    vt = rng.standard_normal((n_t // nu + 1) * nx * ny)
    x = torch.empty(so.size, dtype=torch.float64, device="cuda")
    w = torch.empty_like(x)
    vd = torch.from_numpy(v).cuda()
    _lib.check(lib.pmk_interp_sub_stmv(ctypes.byref(sysd.level_desc()),
                                       ctypes.byref(pair._pair_desc()), _lib.ptr(vd), None,
                                       _lib.ptr(torch.from_numpy(vt).cuda()), _lib.ptr(x),
                                       _lib.ptr(w), _lib.stream_ptr()), "imv")
    xr = v - O.interpolate(po, vt)
    np.testing.assert_array_equal(x.cpu().numpy(), xr)
    np.testing.assert_array_equal(w.cpu().numpy(), O.matvec(so, xr))


def test_reciprocal_division_is_ieee_bitwise():
    """The kernels divide by a vector norm through RN(1/d) and two FMA
    corrections; it must equal IEEE x / d bit for bit, over wide exponent
    ranges, signs, zeros and subnormal-adjacent values."""
    import torch

    from paper_2401_00228_b200 import _lib

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(0)
    n = 1 << 24
    mant = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) + 1.0
    expo = torch.randint(-1000, 1000, (n,), generator=g, device="cuda").to(torch.float64)
    sign = torch.where(torch.rand(n, generator=g, device="cuda") < 0.5, -1.0, 1.0).to(
        torch.float64)
    x = sign * mant * torch.pow(2.0, expo)
    x[:1000] = 0.0
    x[1000:2000] = -0.0
    x[2000:3000] = torch.linspace(1e-310, 1e-300, 1000, device="cuda", dtype=torch.float64)
    out = torch.empty_like(x)
    xh = x.cpu().numpy()
    # reference: numpy's IEEE division (torch divides by a Python scalar on
    # CUDA through a reciprocal multiply, which is not IEEE division)
    for d in (1.0, 3.0, 0.7071067811865476, 123456.789, 1e-3, 2.0 ** -99, 1.2345e20,
              float(np.nextafter(1.0, 2.0)), 9.999999999999999e-1, 0.1, 7.0, 2.0 ** 100):
        _lib.check(lib.pmk_div_check(_lib.ptr(x), d, n, _lib.ptr(out), _lib.stream_ptr()), "div")
        ref = xh / d
        got = out.cpu().numpy()
        same = got.view(np.int64) == ref.view(np.int64)
        assert bool(same.all()), (d, int((~same).sum()))


@pytest.mark.parametrize("nx,ny,n_t,levels", [(300, 20, 32, 3), (520, 37, 16, 3), (40, 333, 32, 4)])
def test_solve_on_split_row_tiles_and_partial_row_tiles(nx, ny, n_t, levels):
    """Full solves whose in-solver march kernels run with rows split into
    several column tiles (nx > 255), row counts that leave a partial last
    6-row / 4-row tile, and non-square grids (dense sine-GEMM coarsest solve),
    against the oracle: iteration count +-1, x <= 1e-10."""
    from oracle import pintmk_oracle as O
    import paper_2401_00228_b200 as P

    rng = np.random.default_rng(nx + ny)
    h = 1.0 / (nx + 1)
    dt = 0.16 * h * h / 3.0
    u0 = rng.standard_normal(nx * ny)
    op = P.build_laplacian(2, nx, ny)
    ops = P.build_step_operators(op, P.ThetaSchemeConfig(0.5, dt, n_t))
    fine = P.FineSystem(ops, u0)
    cfg = P.SolverConfig(tol=1e-8, max_outer=60)
    x, rep = P.multilevel_solve(P.build_hierarchy(fine, levels, ["time"] * (levels - 1), cfg, nu=2))
    oh = O.build(2, nx, ny, 0.5, dt, n_t, u0, levels, ["time"] * (levels - 1),
                 O.Config(tol=1e-8, max_outer=60), nu=2)
    xo, info = O.solve(oh)
    assert abs(rep.outer_iterations - info["iterations"]) <= 1
    assert rel(x, xo) <= 1e-10, rel(x, xo)
