"""BASELINE config 5's literal solver structure at full size: c5_c_dec =
255^2 x 4096 Crank-Nicolson, 5 levels, nu = 2, perturbed decoupled coarsest
level with n_cgs = 256 (one independent solve per coarse slice,
intergrid.py:299-311), FGMRES(30), at the paper's Courant number -- against
the LIVE reference's own run of the same seeded input for a fixed budget of
32 iterations (tests/golden/make_c5c_dec_reference.py: cycle 1 = 30
iterations, then the restart fires and cycle 2 runs 2 more).

North-star bar on the fingerprint: the same iteration count, residual history
within 1e-6 relative (the estimates of both cycles), x within 1e-10 relative
l2 (strided sample and every slice norm), and the true residual.
"""

import os

import numpy as np
import pytest

from tests.cases import BASELINE, gpu_hierarchy

pytestmark = pytest.mark.gpu

FIXTURE = os.path.join(os.path.dirname(__file__), "golden", "c5_c_dec_reference.npz")


@pytest.fixture(scope="module")
def solved():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(FIXTURE):
        pytest.skip("c5_c_dec reference fingerprint not generated")
    from paper_2401_00228_b200 import multilevel_solve

    ref = dict(np.load(FIXTURE))
    case = BASELINE["c5_c_dec"].scaled(max_outer=int(ref["budget"]))
    x, rep = multilevel_solve(gpu_hierarchy(case, u0=torch.from_numpy(case.u0_vector()).cuda()))
    out = {"iters": rep.outer_iterations, "hist": np.array(rep.residual_history),
           "cycles": rep.metadata.get("restart_cycles"),
           "true_res": rep.metadata["true_relative_residual"],
           "x_sub": x[::int(ref["stride"])].cpu().numpy(),
           "slice_norms": torch.linalg.vector_norm(x.reshape(case.n_t + 1, case.m),
                                                   dim=1).cpu().numpy()}
    del x
    torch.cuda.empty_cache()
    return out, ref


def test_restart_fires_and_history_matches(solved):
    ours, ref = solved
    assert ours["iters"] == int(ref["iters"]) == int(ref["budget"])
    assert ours["cycles"] == 2  # 30 + 2: the restart fired once
    np.testing.assert_allclose(ours["hist"], ref["hist"], rtol=1e-6)
    assert abs(ours["true_res"] - float(ref["true_res"])) <= 1e-6 * float(ref["true_res"])


def test_solution_matches_reference(solved):
    ours, ref = solved
    d = np.linalg.norm(ours["x_sub"] - ref["x_sub"]) / np.linalg.norm(ref["x_sub"])
    assert d <= 1e-10, d
    rel = np.abs(ours["slice_norms"] - ref["slice_norms"]) / ref["slice_norms"]
    assert rel.max() <= 1e-10, rel.max()
