"""Time the coarsest solve of a workload in isolation (CUDA events, the
solver's own descriptor), for A/B of the coarsest kernels and ncu captures:

    python tools/coarse_probe.py [case] [reps]
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
c = h.levels[-1]
solver = c.system.diag_factorization
rhs = torch.randn(c.total_dim, dtype=torch.float64, device="cuda")
out = torch.empty_like(rhs)
solver.solve_into(rhs, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    solver.solve_into(rhs, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"case": case.name, "kind": solver.kind, "detail": getattr(solver, "kind_detail", None),
                  "grid": list(c.grid), "slices": c.n_steps + 1, "ms_per_coarse_solve": round(ms, 4),
                  "GB/s_16B_per_elem_per_pass": round(16 * c.total_dim / (ms / 1000) / 1e9, 1),
                  "env": {k: v for k, v in os.environ.items() if k.startswith("PMK_")}}))
