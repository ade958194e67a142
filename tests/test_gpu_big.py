"""A space-time vector longer than 2^31 doubles (17 GB): the 1-D TMA tensor
maps address it with int32 coordinates, so the march kernels switch to plain
bulk copies (64-bit addresses, cp.async.bulk) instead of dropping to the
register kernels.  Checked bitwise against the register kernels
(PMK_MARCH_REG=1, run in a subprocess) on the same seeded input -- both are
bitwise the reference's matvec (tests/test_gpu_parity.py at small sizes).
Also: the bulk path (PMK_TMA_BULK=1) on the small golden cases, bitwise.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2401_00228_b200 as P
nx, steps = 255, 33026           # (steps + 1) * 255^2 = 2.1475e9 > 2^31
op = P.build_laplacian(2, nx, nx)
ops = P.build_step_operators(op, P.ThetaSchemeConfig(0.5, 1e-5, steps))
sysm = P.BlockBidiagonalSystem(ops.psi, ops.phi, steps, grid=(nx, nx), dim=2,
                               spectral=ops.spectral_info)
N = (steps + 1) * nx * nx
g = torch.Generator(device="cuda").manual_seed(11)
v = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
out = torch.empty_like(v)
sysm.matvec_into(v, out)  # (warm-up)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sysm.matvec_into(v, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
del v
sums = out.view(steps + 1, nx * nx).sum(dim=1)
sample = out[::1000003]
print(json.dumps({"N": N, "sums": sums.cpu().tolist(), "sample": sample.cpu().tolist(),
                  "last": out[-nx * nx:].sum().item(), "ms": ms, "GBps": 16.0 * N / ms / 1e6}))
"""


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    free, _ = torch.cuda.mem_get_info()
    if free < 40e9:
        pytest.skip("needs ~40 GB of free device memory")


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    proc = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True,
                          text=True, timeout=900)
    assert proc.returncode == 0, proc.stderr[-2000:]
    out = json.loads(proc.stdout.strip().splitlines()[-1])
    out["stderr"] = proc.stderr
    return out


def test_matvec_beyond_int32_coordinates_bitwise():
    tma = _run({"PMK_DEBUG": "1"})
    reg = _run({"PMK_MARCH_REG": "1"})
    assert tma["N"] >= 2**31
    assert "[pmk] tma mode 0" in tma["stderr"] and "bulk 1" in tma["stderr"]  # TMA, bulk copies
    print(f"K-MV at N = {tma['N']}: TMA bulk {tma['ms']:.2f} ms ({tma['GBps']:.0f} GB/s), "
          f"register path {reg['ms']:.2f} ms ({reg['GBps']:.0f} GB/s)")
    np.testing.assert_array_equal(np.array(tma["sums"]), np.array(reg["sums"]))
    np.testing.assert_array_equal(np.array(tma["sample"]), np.array(reg["sample"]))
    assert tma["last"] == reg["last"]


def test_bulk_copy_path_bitwise_on_golden_cases():
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x",
                           os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                           "-k", "matvec_bitwise or transfers_bitwise or fused_kernels or "
                                 "solve_parity"],
                          env=dict(os.environ, PMK_TMA_BULK="1"), capture_output=True, text=True,
                          timeout=1200, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout[-3000:]


def test_dst_gemm_coarsest_beyond_grid_dimension_limits():
    """The sine-GEMM coarsest path (n + 1 not a power of two) on 100^2 x
    42000 slices: (slices x 100) / 64 M-tiles exceed the 65535 gridDim.y limit
    that round 1's GEMM launch put them in.  Size-independent property: the
    forward substitution inverts the block system, A (A^{-1} r) = r."""
    import torch

    import paper_2401_00228_b200 as P

    n, steps = 100, 41999
    op = P.build_laplacian(2, n, n)
    ops = P.build_step_operators(op, P.ThetaSchemeConfig(0.5, 2e-5, steps))
    fine = P.FineSystem(ops, torch.zeros(n * n, dtype=torch.float64, device="cuda"))
    assert fine.diag_factorization.kind_detail == "dst-gemm"
    g = torch.Generator(device="cuda").manual_seed(3)
    r = torch.randn((steps + 1) * n * n, dtype=torch.float64, device="cuda", generator=g)
    u = fine.forward_solve(r)
    back = fine.matvec(u)
    err = (torch.linalg.vector_norm(back - r) / torch.linalg.vector_norm(r)).item()
    assert err <= 1e-12, err


def test_tall_tile_matvec_is_bitwise_the_oracle_matvec():
    """Vectors of >= 2^25 doubles on grids with >= 64 rows take the 16-row
    matvec tile (csrc/pmk_march_tma.cu, PMK_MV_CFG): bitwise equal to the
    oracle's (= the reference's) matvec on 127^2 x 2101 slices, with dropped
    rows, and on an odd row count that leaves a partial last tile (120)."""
    from oracle import pintmk_oracle as O
    import paper_2401_00228_b200 as P

    for nx, ny, steps, dropped in ((127, 127, 2100, (3, 700, 2100)), (150, 120, 1900, ())):
        op = P.build_laplacian(2, nx, ny)
        ops = P.build_step_operators(op, P.ThetaSchemeConfig(0.5, 1e-5, steps))
        sysm = P.BlockBidiagonalSystem(ops.psi, ops.phi, steps, dropped=dropped, grid=(nx, ny),
                                       dim=2, spectral=ops.spectral_info)
        assert (steps + 1) * nx * ny >= 1 << 25
        v = np.random.default_rng(5).standard_normal((steps + 1) * nx * ny)
        a = O.laplacian(2, nx, ny)[0]
        d, b = O.blocks_from(a, 0.5, 1e-5)
        want = O.matvec(O.System(d, b, steps, dropped), v)
        np.testing.assert_array_equal(sysm.matvec(v), want)
