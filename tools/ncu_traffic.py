"""From an ncu launch list (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum; --print-kernel-base demangled) write the per-category
DRAM traffic per launch that bench.py reports as roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/launches.csv > profiles/ncu_traffic.json
"""

import collections
import csv
import json
import re
import sys

CATS = [(r"march_tma(?:_1d)?_kernel<(?:\(int\))?0", "march_mv"),
        (r"march_(?:tma(?:_1d)?|lean)_kernel<(?:\(int\))?1", "march_mvr"),
        (r"march_(?:tma(?:_1d)?|lean)_kernel<(?:\(int\))?2", "march_imv"),
        (r"mgs_pass|icwy_dots|icwy_update", "mgs_pass"),
        (r"dot_partials|diffsq_partials", "reduce"), (r"assemble", "assemble"),
        (r"dst_rows|dst_cols", "coarse_dst"),
        (r"dgemm", "coarse_gemm"),
        (r"dst_recurrence|rec_chunk", "coarse_recurrence"), (r"copy_row", "coarse_misc")]


def category(name: str):
    for key, cat in CATS:
        if re.search(key, name):
            return cat
    return None


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    idx = {h: i for i, h in enumerate(rows[hi])}
    scale_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.defaultdict(lambda: {"launches": set(), "bytes": 0.0})
    for r in rows[hi + 1:]:
        if len(r) < len(idx):
            continue
        cat = category(r[idx["Kernel Name"]])
        if not cat or not r[idx["Metric Name"]].startswith("dram__bytes"):
            continue
        v = float(r[idx["Metric Value"]].replace(",", "")) * scale_b.get(r[idx["Metric Unit"]], 1)
        per[cat]["launches"].add(r[idx["ID"]])
        per[cat]["bytes"] += v
    out = {c: d["bytes"] / len(d["launches"]) for c, d in per.items() if d["launches"]}
    out["_source"] = path
    out["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu, "
                    "serialised launches of one full c5_c solve); compare with the "
                    "algorithmic bytes_per_launch of bench.py's roofline")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
