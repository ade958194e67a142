"""Mid-size parity against fingerprints of the LIVE reference
(tests/golden/make_golden.py --mid): realistic agglomerated coarsest levels
(the EIG coarsest solve -- separable eigen-transforms, per-mode recurrence,
the cluster chain kernel for the odd-grid B^T coupling), the default "auto"
schedule where the stability screen inserts space moves, the spatial
coarsening switch at the end of a time hierarchy on 127^2 and 255^2 grids,
and a caller's own row-scaled operator whose coarsest level takes the LINE
(2-D, 16129 unknowns per slice, past the dense-inverse limit) and PCR (1-D,
32 decoupled chains) kinds by default.

Bars: coarsest forward_solve <= 1e-12 relative (rounding: eigen-transforms vs
the reference's SuperLU / Thomas), apply_preconditioner <= 1e-10, full solve
(or fixed budget when the reference does not converge) iteration count +-1,
residual history rtol 1e-6, x <= 1e-10 relative on the fingerprint.
"""

import os

import numpy as np
import pytest

from tests.cases import MID, fingerprint, gpu_hierarchy, mid_inputs

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# cases whose coarsest level takes a kind from csrc/pmk_lines.cu by default
DEFAULT_KIND = {"line_mid": "line", "line_dec_mid": "line", "line_255_mid": "line",
                "pcr_dec_mid": "pcr"}


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _fixture(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} fingerprint not generated")
    return dict(np.load(path))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", sorted(MID))
def test_mid_parity(name):
    import torch

    from paper_2401_00228_b200 import apply_preconditioner, multilevel_solve

    g = _fixture(name)
    case = MID[name]
    h = gpu_hierarchy(case)
    assert list(h.moves) == [str(m) for m in g["moves"]]
    lv = h.levels
    coarse = lv[-1].system.diag_factorization
    if any(m in ("space", "time_space") for m in h.moves):
        assert coarse.kind == "eig", coarse.kind
    if name in DEFAULT_KIND:
        assert coarse.kind == DEFAULT_KIND[name], coarse.kind
    cs_in, pc_in = mid_inputs(case, (lv[-1].total_dim, lv[0].total_dim))
    cs = lv[-1].system.forward_solve(torch.from_numpy(cs_in).cuda()).cpu().numpy()
    f = fingerprint(cs, lv[-1].n_steps + 1)
    assert rel(f["sub"], g["cs_sub"]) <= 1e-12, rel(f["sub"], g["cs_sub"])
    assert rel(f["norms"], g["cs_norms"]) <= 1e-12
    pc = apply_preconditioner(h, 0, torch.from_numpy(pc_in).cuda()).cpu().numpy()
    f = fingerprint(pc, lv[0].n_steps + 1)
    assert rel(f["sub"], g["pc_sub"]) <= 1e-10, rel(f["sub"], g["pc_sub"])
    x, rep = multilevel_solve(h)
    assert abs(rep.outer_iterations - int(g["iters"])) <= 1
    n = min(len(rep.residual_history), len(g["hist"]))
    np.testing.assert_allclose(rep.residual_history[:n], g["hist"][:n], rtol=1e-6)
    f = fingerprint(x, lv[0].n_steps + 1)
    assert rel(f["sub"], g["x_sub"]) <= 1e-10, rel(f["sub"], g["x_sub"])
    assert rel(f["norms"], g["x_norms"]) <= 1e-10
