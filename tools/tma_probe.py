"""Probe the TMA march path on small shapes (blocking launches)."""
import ctypes, os, sys
os.environ["CUDA_LAUNCH_BLOCKING"] = "1"
os.environ["PMK_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2401_00228_b200 import _lib
lib = _lib.load()
def run(dim, nx, ny, n_steps):
    d = _lib.LevelDesc(); d.dim, d.nx, d.ny, d.n_steps = dim, nx, ny, n_steps
    for st, vals in ((d.diag_t, (-1, -1, 5, -1, -1)), (d.sub_t, (0.5, 0.5, 1, 0.5, 0.5))):
        st.var = 0
        for i, v in enumerate(vals): st.c[i] = v
    N = (n_steps + 1) * nx * ny
    v = torch.randn(N, dtype=torch.float64, device="cuda"); out = torch.zeros_like(v)
    rc = lib.pmk_stmv(ctypes.byref(d), _lib.ptr(v), _lib.ptr(out), _lib.stream_ptr())
    print("RESULT", dim, nx, ny, n_steps, "rc", rc, flush=True)
    return rc
case = sys.argv[1].split(",")
run(int(case[0]), int(case[1]), int(case[2]), int(case[3]))
