"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes])
into a per-kernel markdown table: launches, total ms, share, DRAM GB, GB/s.

    python tools/ncu_summary.py gpurun_out/launches.csv > profiles/rN_launches.md
"""

import collections
import csv
import math
import re
import sys


def short_name(name: str) -> str:
    m = re.search(r"march_tma_kernel<(?:\(int\))?(\d), (?:\(int\))?(\d)", name)
    if m:
        return {"0": "march_mv", "1": "march_mvr", "2": "march_imv"}[m.group(1)] + f"[{m.group(2)}d]"
    m = re.search(r"march_lean_kernel<(?:\(int\))?(\d)", name)
    if m:
        return {"1": "march_mvr", "2": "march_imv"}[m.group(1)] + "[2d]"
    m = re.search(r"march_tma_1d_kernel<(?:\(int\))?(\d)", name)
    if m:
        return {"0": "march_mv", "1": "march_mvr", "2": "march_imv"}[m.group(1)] + "[1d]"
    base = re.sub(r"\(.*", "", name)
    base = base.split("::")[-1]
    return re.sub(r"<.*", "", base) or name[:40]


def main(path: str) -> None:
    rows = [r for r in csv.reader(open(path)) if r]
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    idx = {h: i for i, h in enumerate(hdr)}
    scale_t = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
               "msecond": 1.0, "s": 1e3, "second": 1e3}
    scale_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    launches = collections.OrderedDict()  # ID -> [name, ms, bytes]
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        try:
            v = float(r[idx["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        rec = launches.setdefault(r[idx["ID"]], [short_name(r[idx["Kernel Name"]]), 0.0, 0.0])
        met, unit = r[idx["Metric Name"]], r[idx["Metric Unit"]]
        if met == "gpu__time_duration.sum":
            rec[1] += v * scale_t.get(unit, 1e-6)
        elif met.startswith("dram__bytes"):
            rec[2] += v * scale_b.get(unit, 1.0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    by_size = collections.defaultdict(lambda: [0, 0.0, 0.0])
    total = 0.0
    for name, ms, b in launches.values():
        for a_, key in ((agg, name), (by_size, (name, size_bucket(b)))):
            a_[key][0] += 1
            a_[key][1] += ms
            a_[key][2] += b
        total += ms
    print(f"Kernel time per launch list (serialised, cold): total {total:.1f} ms\n")
    print("| kernel | launches | ms | share | DRAM GB | DRAM GB/s |")
    print("|---|---:|---:|---:|---:|---:|")
    for k, (n, ms, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = b / 1e9 / (ms / 1e3) if ms and b else 0.0
        print(f"| {k} | {n} | {ms:.2f} | {100 * ms / total:.1f}% | {b / 1e9:.1f} | {gbs:.0f} |")
    print("\nBy DRAM bytes per launch (a proxy for the hierarchy level):\n")
    print("| kernel | bytes/launch | launches | ms | us/launch | DRAM GB/s |")
    print("|---|---|---:|---:|---:|---:|")
    for (k, bk), (n, ms, b) in sorted(by_size.items(), key=lambda x: -x[1][1]):
        if ms < 0.01 * total:
            continue
        gbs = b / 1e9 / (ms / 1e3) if ms and b else 0.0
        print(f"| {k} | {bk} | {n} | {ms:.2f} | {1e3 * ms / n:.1f} | {gbs:.0f} |")


def size_bucket(b: float) -> str:
    if b <= 0:
        return "0"
    e = int(math.floor(math.log2(b)))
    lo = 2.0 ** e
    for unit, f in (("GB", 1e9), ("MB", 1e6), ("KB", 1e3)):
        if lo >= f:
            return f"[{lo / f:.3g}, {2 * lo / f:.3g}) {unit}"
    return f"[{lo:.0f}, {2 * lo:.0f}) B"


if __name__ == "__main__":
    main(sys.argv[1])
