"""Loss of orthogonality of the FGMRES basis (one-reduce MGS on the device vs
the reference's MGS in the oracle) and the Arnoldi relation, per case.

    python tools/orth_probe.py [case ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import pintmk_oracle as O  # noqa: E402
from paper_2401_00228_b200 import fgmres  # noqa: E402
from tests.cases import BASELINE, SMALL, gpu_hierarchy, oracle_hierarchy  # noqa: E402


def loss(basis):
    V = np.stack(basis, axis=1)
    return float(np.abs(V.T @ V - np.eye(V.shape[1])).max())


def main(names):
    for name in names:
        case = SMALL.get(name) or BASELINE[name]
        h = gpu_hierarchy(case)
        oh = oracle_hierarchy(case)
        rhs = oh.rhs.ravel()
        it = 12
        _, rep = fgmres(h, 0, rhs, tol=None, max_iter=it, keep_basis=True)
        _, info = O.fgmres(oh, 0, rhs, None, it, keep_basis=True)
        md = rep.metadata
        n = len(md["preconditioned"])
        Z = np.stack(md["preconditioned"], axis=1)
        V = np.stack(md["basis"][:n + 1], axis=1)
        AZ = np.stack([O.matvec(oh.fine, Z[:, j]) for j in range(n)], axis=1)
        arn = np.linalg.norm(AZ - V @ md["hessenberg"]) / np.linalg.norm(AZ)
        print(f"{name}: n={n} loss gpu(ICWY) {loss(md['basis']):.3e}  oracle(MGS) "
              f"{loss(info['basis']):.3e}  arnoldi {arn:.2e}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3_small", "c5_small", "mid_2d"])
