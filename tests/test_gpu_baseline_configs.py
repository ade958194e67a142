"""GPU vs CPU oracle on the BASELINE.json shapes themselves.

* Literal configs 1-4 (Courant numbers 24-512, where the reference MLK
  stagnates) are compared at a fixed iteration budget:
  same number of iterations, residual histories within 1e-6 relative, and
  the iterates x_K (the residual estimate is flat there, so the Hessenberg
  least-squares problem is ill-conditioned: x is held to 1e-8 relative).
* Regime-adjusted companions (same shapes at the paper's Courant number)
  converge, and are held to the north-star bar: same iteration count (+-1)
  and x within 1e-10 relative l2.  (The config-4 companion, TS x TS nu = 4
  at theta = 1, still needs more than 200 iterations in the reference -- true
  residual 1.5e-8 after 200 -- so config 4 is covered at a fixed budget.)
Config 5 (2.7e8 unknowns, 2.1 GB vectors) costs the CPU oracle minutes per
iteration: one iteration is compared here; the converged full-size solve is
covered by the bench's true-residual check and the shrunk c5 cases.
"""

import numpy as np
import pytest

from tests.cases import BASELINE, gpu_hierarchy, oracle_hierarchy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rel(a, b):
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _run_both(case):
    from oracle import pintmk_oracle as O
    from paper_2401_00228_b200 import multilevel_solve

    x, rep = multilevel_solve(gpu_hierarchy(case))
    xo, info = O.solve(oracle_hierarchy(case))
    return x, rep, xo, info


@pytest.mark.parametrize("name,budget", [("c1", 60), ("c2", 10), ("c3", 20), ("c4", 10),
                                         ("c5", 1)])
def test_literal_config_fixed_budget(name, budget):
    case = BASELINE[name].scaled(max_outer=budget)
    x, rep, xo, info = _run_both(case)
    assert rep.outer_iterations == info["iterations"] == budget
    np.testing.assert_allclose(rep.residual_history, info["history"], rtol=1e-6)
    assert rel(x, xo) <= 1e-8, rel(x, xo)


@pytest.mark.parametrize("name", ["c1_c", "c2_c", "c3_c"])
def test_companion_full_solve(name):
    case = BASELINE[name]
    x, rep, xo, info = _run_both(case)
    assert rep.converged and info["converged"]
    assert abs(rep.outer_iterations - info["iterations"]) <= 1
    assert rel(x, xo) <= 1e-10, rel(x, xo)
