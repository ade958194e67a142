"""Throughput of the coarsest transforms' fp64 GEMM (pmk_dgemm: DMMA tensor
cores; PMK_GEMM=simt: CUDA-core kernel) on the EIG / DST-GEMM shapes.

    python tools/gemm_probe.py        (on the GPU box)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_00228_b200 import _lib  # noqa: E402

lib = _lib.load()
out = {}
for (m, n, k, batch) in [(65 * 127, 127, 127, 1), (127, 127, 127, 65), (257 * 255, 255, 255, 1),
                         (255, 255, 255, 257), (8192, 8192, 8192, 1)]:
    a = torch.randn(batch * m * k, dtype=torch.float64, device="cuda")
    b = torch.randn(batch * k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(batch * m * n, dtype=torch.float64, device="cuda")
    sa = m * k if batch > 1 else 0
    sb = k * n if batch > 1 else 0
    args = (m, n, k, _lib.ptr(a), k, sa, _lib.ptr(b), n, sb, _lib.ptr(c), n, m * n, batch)
    for _ in range(2):
        lib.pmk_dgemm(*args, _lib.stream_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        lib.pmk_dgemm(*args, _lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * m * n * k * batch / (ms / 1000.0) / 1e12
    out[f"{m}x{n}x{k}x{batch}"] = {"ms": round(ms, 4), "TFLOP/s": round(tf, 2)}
print(json.dumps({"impl": os.environ.get("PMK_GEMM", "dmma"), "gemm": out}))
