"""Time the plain space-time matvec (pmk_stmv, BlockBidiagonalSystem.matvec)
alone on a workload's fine vector: CUDA events around back-to-back launches.

    PMK_MV_CFG=<n> python tools/mv_probe.py [case] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tests.cases import BASELINE, MID, gpu_hierarchy  # noqa: E402

case = {**MID, **BASELINE}[sys.argv[1] if len(sys.argv) > 1 else "c5_c"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = gpu_hierarchy(case, u0=torch.from_numpy(case.u0_vector()).cuda())
sysm = h.levels[0].system
v = torch.randn(h.levels[0].total_dim, dtype=torch.float64, device="cuda")
out = torch.empty_like(v)
for _ in range(3):
    sysm.matvec_into(v, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    sysm.matvec_into(v, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"case": case.name, "cfg": os.environ.get("PMK_MV_CFG", "0"),
                  "ms_per_matvec": round(ms, 4),
                  "GB/s": round(16.0 * v.numel() / (ms / 1e3) / 1e9, 1)}))
