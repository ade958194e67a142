"""The headline workload c5_c (255^2 x 4096 Crank-Nicolson, 5 levels, nu = 2,
exact coarsest chain, FGMRES(30), tol 1e-8; 2.66e8 unknowns) against the
LIVE reference's own solve of the same seeded input, recorded by
tests/golden/make_c5c_reference.py (about an hour of CPU there, so it is a
committed fingerprint, not a per-run oracle call).

North-star bar: the same iteration count (+-1) and x within 1e-10 relative
l2 -- checked on x at a fixed stride (65k entries spread over every time
slice) and on the l2 norm of every one of the 4097 time slices.
"""

import os

import numpy as np
import pytest

from tests.cases import BASELINE, gpu_hierarchy

pytestmark = pytest.mark.gpu

FIXTURE = os.path.join(os.path.dirname(__file__), "golden", "c5_c_reference.npz")


@pytest.fixture(scope="module")
def solved():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(FIXTURE):
        pytest.skip("c5_c reference fingerprint not generated")
    from paper_2401_00228_b200 import multilevel_solve

    case = BASELINE["c5_c"]
    x, rep = multilevel_solve(gpu_hierarchy(case, u0=torch.from_numpy(case.u0_vector()).cuda()))
    ref = dict(np.load(FIXTURE))
    out = {"iters": rep.outer_iterations, "hist": np.array(rep.residual_history),
           "true_res": rep.metadata["true_relative_residual"],
           "x_sub": x[::int(ref["stride"])].cpu().numpy(),
           "slice_norms": torch.linalg.vector_norm(x.reshape(case.n_t + 1, case.m),
                                                   dim=1).cpu().numpy()}
    del x
    torch.cuda.empty_cache()
    return out, ref


def test_headline_iterations_and_residual(solved):
    ours, ref = solved
    assert abs(ours["iters"] - int(ref["iters"])) <= 1
    assert ours["true_res"] <= 1e-8 and float(ref["true_res"]) <= 1e-8
    n = min(len(ours["hist"]), len(ref["hist"]))
    np.testing.assert_allclose(ours["hist"][:n], ref["hist"][:n], rtol=1e-6)


def test_headline_solution_matches_reference(solved):
    ours, ref = solved
    d = np.linalg.norm(ours["x_sub"] - ref["x_sub"]) / np.linalg.norm(ref["x_sub"])
    assert d <= 1e-10, d
    rel = np.abs(ours["slice_norms"] - ref["slice_norms"]) / ref["slice_norms"]
    assert rel.max() <= 1e-10, rel.max()
