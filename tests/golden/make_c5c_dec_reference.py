"""Fingerprint of the LIVE reference on BASELINE config 5's literal solver
structure at the paper's Courant number: c5_c_dec = 255^2 x 4096
Crank-Nicolson, 5 levels, nu = 2, perturbed decoupled coarsest level with
n_cgs = 256 (one independent solve per coarse time slice,
intergrid.py:299-311, solver.py:209-213), FGMRES(30) through the restart
wrapper of SURVEY.md section 8(c) around the reference's own fgmres
(solver.py:362-456), for a FIXED budget of 32 outer iterations, so the
restart fires once (cycle 1: 30 iterations, cycle 2: 2).  For
tests/test_gpu_c5_dec.py.

    python tests/golden/make_c5c_dec_reference.py [basis_dir] [ram_vectors]

Storage, not arithmetic: cycle 1 keeps 61 Krylov vectors of 2.13 GB
(basis + preconditioned, solver.py:385-388) = 130 GB, more than this
container's free disk.  The reference's `_VectorStore` (solver.py:268-298)
is swapped for a split store that keeps the first `ram_vectors` fine-level
vectors in RAM and the rest in the reference's own unlinked-memmap layout.
Every floating-point operation is the reference's; only where the bytes
sit changes (a store returns the same float64 values it was given).

x itself is too large to commit; like make_c5c_reference.py the fixture
holds the iteration count, residual history, true residual, slice norms
and x at a fixed stride.
"""

from __future__ import annotations

import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import make_golden as G  # noqa: E402  (imports the reference from /root/reference)

from tests.cases import BASELINE  # noqa: E402

STRIDE = 4099
BUDGET = 32
_ram_left = [0]
_fine_dim = [0]
_Orig = G.R_sol._VectorStore


class SplitStore:
    """Drop-in for the reference's _VectorStore (same methods); fine-level
    vectors go to RAM while the quota lasts, the rest to a disk memmap."""

    def __init__(self, dim, capacity, use_disk, directory=None):
        self._split = dim == _fine_dim[0]
        if not self._split:
            self._inner = _Orig(dim, capacity, use_disk, directory)
            return
        self._ram: list[np.ndarray] = []
        self._file = tempfile.TemporaryFile(dir=directory)
        self._mm = np.memmap(self._file, dtype=np.float64, mode="w+", shape=(capacity, dim))
        self._where: list[tuple[bool, int]] = []
        self._n_disk = 0

    def append(self, vec):
        if not self._split:
            return self._inner.append(vec)
        if _ram_left[0] > 0:
            _ram_left[0] -= 1
            self._where.append((True, len(self._ram)))
            self._ram.append(np.array(vec, copy=True))
        else:
            self._mm[self._n_disk] = vec
            self._where.append((False, self._n_disk))
            self._n_disk += 1

    def __getitem__(self, j):
        if not self._split:
            return self._inner[j]
        ram, k = self._where[j]
        return self._ram[k] if ram else self._mm[k]

    def close(self):
        if not self._split:
            return self._inner.close()
        _ram_left[0] += len(self._ram)
        self._ram.clear()
        del self._mm
        self._file.close()


def main():
    basis_dir = sys.argv[1] if len(sys.argv) > 1 else "/tmp/c5cdec_basis"
    _ram_left[0] = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    os.makedirs(basis_dir, exist_ok=True)
    case = BASELINE["c5_c_dec"].scaled(max_outer=BUDGET)
    _fine_dim[0] = case.N
    G.R_sol._VectorStore = SplitStore
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
        "wall_s": np.array(wall), "budget": np.array(BUDGET),
    }
    path = os.path.join(HERE, "c5_c_dec_reference.npz")
    np.savez_compressed(path, **out)
    print(f"c5_c_dec: iters={total} true_res={true_res:.3e} wall={wall:.0f} s "
          f"hist[-1]={hist[-1]:.3e} -> {os.path.getsize(path) / 1024:.0f} KiB", flush=True)


if __name__ == "__main__":
    main()
