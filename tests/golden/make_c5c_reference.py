"""Fingerprint of the LIVE reference's solve of the headline workload c5_c
(255^2 x 4096 Crank-Nicolson, 5 levels, nu = 2, exact coarsest chain,
FGMRES(30) via the restart wrapper of SURVEY.md section 8(c), tol 1e-8),
for tests/test_gpu_headline.py.  Run here, where /root/reference exists; the
fixture travels, the reference does not.  About an hour of CPU and ~85 GB of
basis spill (the reference's own _VectorStore memmap, basis_dir below).

    python tests/golden/make_c5c_reference.py [basis_dir]

x itself (2.13 GB) is too large to commit; the fixture holds the iteration
count, the residual history, the true residual, the l2 norm of every time
slice of x, and x at a fixed stride (every 4099th entry, 65k values).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import make_golden as G  # noqa: E402  (imports the reference from /root/reference)

from tests.cases import BASELINE  # noqa: E402

STRIDE = 4099


def main():
    basis_dir = sys.argv[1] if len(sys.argv) > 1 else "/tmp/c5c_basis"
    os.makedirs(basis_dir, exist_ok=True)
    case = BASELINE["c5_c"]
    t0 = time.time()
    hier = G.reference_hierarchy(case)
    hier.config.basis_dir = basis_dir
    print(f"hierarchy built in {time.time() - t0:.0f} s", flush=True)
    t1 = time.time()
    x, total, hist = G.reference_restarted(hier, case.tol, case.max_outer, case.restart)
    wall = time.time() - t1
    true_res = float(hier.fine.relative_residual(x))
    xs = x.reshape(case.n_t + 1, case.m)
    out = {
        "iters": np.array(total), "hist": np.array(hist), "true_res": np.array(true_res),
        "slice_norms": np.linalg.norm(xs, axis=1), "norm": np.array(np.linalg.norm(x)),
        "stride": np.array(STRIDE), "x_sub": np.ascontiguousarray(x[::STRIDE]),
        "wall_s": np.array(wall),
    }
    path = os.path.join(HERE, "c5_c_reference.npz")
    np.savez_compressed(path, **out)
    print(f"c5_c: iters={total} true_res={true_res:.3e} wall={wall:.0f} s "
          f"-> {os.path.getsize(path) / 1024:.0f} KiB", flush=True)


if __name__ == "__main__":
    main()
