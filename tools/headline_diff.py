"""Measured distance of the c5_c GPU solve from the live reference's
(tests/golden/c5_c_reference.npz): iterations, residual history, x at a
fixed stride, per-slice norms.

    python tools/headline_diff.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_00228_b200 import multilevel_solve  # noqa: E402
from tests.cases import BASELINE, gpu_hierarchy  # noqa: E402

ref = dict(np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests", "golden", "c5_c_reference.npz")))
case = BASELINE["c5_c"]
x, rep = multilevel_solve(gpu_hierarchy(case, u0=torch.from_numpy(case.u0_vector()).cuda()))
xs = x[::int(ref["stride"])].cpu().numpy()
sn = torch.linalg.vector_norm(x.reshape(case.n_t + 1, case.m), dim=1).cpu().numpy()
h = np.array(rep.residual_history)
print(f"iterations ours {rep.outer_iterations} reference {int(ref['iters'])}")
print(f"true residual ours {rep.metadata['true_relative_residual']:.6e} "
      f"reference {float(ref['true_res']):.6e}")
print(f"residual history max rel diff {np.max(np.abs(h - ref['hist']) / ref['hist']):.3e}")
print(f"x (every {int(ref['stride'])}th entry) rel l2 diff "
      f"{np.linalg.norm(xs - ref['x_sub']) / np.linalg.norm(ref['x_sub']):.3e}")
print(f"slice norms max rel diff {np.max(np.abs(sn - ref['slice_norms']) / ref['slice_norms']):.3e}")
print(f"||x|| ours {torch.linalg.vector_norm(x).item():.15e} reference {float(ref['norm']):.15e}")
