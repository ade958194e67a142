"""GPU idle gaps inside one c5_c solve: kernel start/end timestamps from the
torch profiler (CUPTI activity trace), busy time vs wall time, and the
largest gaps with the kernels around them.

    python tools/gap_probe.py [case]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2401_00228_b200 import multilevel_solve  # noqa: E402
from tests.cases import BASELINE, gpu_hierarchy  # noqa: E402


def main():
    case = BASELINE[sys.argv[1] if len(sys.argv) > 1 else "c5_c"]
    h = gpu_hierarchy(case, u0=torch.from_numpy(case.u0_vector()).cuda())
    for _ in range(2):
        multilevel_solve(h)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        multilevel_solve(h)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
          and e.time_range.elapsed_us() >= 0]
    ev.sort(key=lambda e: e.time_range.start)
    ev = [e for e in ev if "Memcpy" not in e.name and "Memset" not in e.name] or ev
    t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
    busy, last_end, gaps = 0.0, t0, []
    for e in ev:
        s, f = e.time_range.start, e.time_range.end
        if s > last_end:
            gaps.append((s - last_end, e.name[:50]))
        busy += max(0.0, f - max(s, last_end))
        last_end = max(last_end, f)
    wall = t1 - t0
    print(f"kernels {len(ev)}  wall {wall / 1e3:.1f} ms  busy {busy / 1e3:.1f} ms  "
          f"idle {(wall - busy) / 1e3:.1f} ms ({(wall - busy) / wall:.1%})")
    gaps.sort(reverse=True)
    hist = {}
    for g, _ in gaps:
        b = "<2us" if g < 2 else "<5us" if g < 5 else "<20us" if g < 20 else "<100us" if g < 100 \
            else ">=100us"
        hist[b] = hist.get(b, [0, 0.0])
        hist[b][0] += 1
        hist[b][1] += g
    for b in ["<2us", "<5us", "<20us", "<100us", ">=100us"]:
        if b in hist:
            print(f"  gaps {b:>7}: {hist[b][0]:5d}  total {hist[b][1] / 1e3:.2f} ms")
    for g, n in gaps[:12]:
        print(f"  {g:8.1f} us before {n}")
    st = torch.cuda.memory_stats()
    print("allocator: segments allocated", st.get("segment.all.allocated"),
          "freed", st.get("segment.all.freed"), "alloc retries", st.get("num_alloc_retries"),
          "device mallocs", st.get("num_device_alloc"), "frees", st.get("num_device_free"))


if __name__ == "__main__":
    main()
