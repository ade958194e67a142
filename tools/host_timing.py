"""Host-side timing of the outer FGMRES loop (where does non-kernel time go?)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2401_00228_b200 import _lib, solver as S
from tests.cases import BASELINE, gpu_hierarchy
case = BASELINE[sys.argv[1] if len(sys.argv) > 1 else "c5_c"]
h = gpu_hierarchy(case, u0=torch.from_numpy(case.u0_vector()).cuda())
S.multilevel_solve(h)  # warm
lib = _lib.load(); s = _lib.stream_ptr(); H = h._native
lvl, nxt = h.levels[0], h.levels[1]
b = h.fine.rhs.reshape(-1)
torch.cuda.synchronize()
T0 = time.perf_counter()
lib.pmk_fgmres_begin(H, 0, _lib.ptr(b), 200, 1e-8, s)
st = S._state(h, 0)
w = S._empty(lvl.total_dim); vs = []; cos = []
tl = []; ts = []; tg = []
for j in range(40):
    t0 = time.perf_counter()
    v = S._empty(lvl.total_dim); co = S._empty(nxt.total_dim); vs.append(v); cos.append(co)
    t1 = time.perf_counter()
    lib.pmk_fgmres_step(H, 0, j, _lib.ptr(v), _lib.ptr(w), _lib.ptr(co), s)
    t2 = time.perf_counter()
    st = S._state(h, 0)
    t3 = time.perf_counter()
    tl.append((t1 - t0) * 1e3); tg.append((t2 - t1) * 1e3); ts.append((t3 - t2) * 1e3)
    if st["rel"] <= 1e-8: break
x = S._empty(lvl.total_dim)
lib.pmk_fgmres_finish(H, 0, _lib.ptr(x), s); torch.cuda.synchronize()
T1 = time.perf_counter()
print("iterations", j + 1, "total %.1f ms" % ((T1 - T0) * 1e3))
print("alloc ms", ["%.2f" % v for v in tl])
print("enqueue ms", ["%.2f" % v for v in tg])
print("sync ms", ["%.2f" % v for v in ts])
