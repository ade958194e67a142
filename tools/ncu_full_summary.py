"""Summarise `ncu --set full` captures (one kernel each) into a markdown table:
duration, DRAM and L1 throughput, issue activity, occupancy, registers, DRAM
bytes, and the warp-stall breakdown from the SASS source page.

    python tools/ncu_full_summary.py gpurun_out/r1_*.ncu-rep > profiles/r1_ncu_full.md
"""
import csv
import io
import subprocess
import sys

METRICS = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
           "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
           "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
           "Block Limit Registers", "Block Limit Shared Mem"]


def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    name, vals = None, {}
    for r in rows[1:]:
        if len(r) <= ix["Metric Value"]:
            continue
        name = r[ix["Kernel Name"]]
        m = r[ix["Metric Name"]]
        if m in METRICS and m not in vals:
            vals[m] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    return name, vals


def stalls(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {r: 0 for r in reasons}
    insts = 0
    for r in rows[2:]:
        for x in reasons:
            try:
                tot[x] += int(r[ix[x]] or 0)
            except (ValueError, IndexError):
                pass
        try:
            insts += int(r[ix["Instructions Executed"]].replace(",", ""))
        except (ValueError, IndexError, KeyError):
            pass
    T = sum(tot.values()) or 1
    top = sorted(tot.items(), key=lambda t: -t[1])[:4]
    return ", ".join(f"{k[6:]} {v / T:.0%}" for k, v in top), insts


def main(paths):
    print("| capture | kernel | " + " | ".join(METRICS) + " | warp instructions | top stalls |")
    print("|---" * (len(METRICS) + 4) + "|")
    for p in paths:
        name, vals = details(p)
        st, insts = stalls(p)
        short = name.split("(")[0].split("::")[-1][:60] if name else "?"
        cells = [f"{vals[m][0]} {vals[m][1]}".strip() if m in vals else "" for m in METRICS]
        print(f"| {p.split('/')[-1]} | `{short}` | " + " | ".join(cells) +
              f" | {insts:,} | {st} |")


if __name__ == "__main__":
    main(sys.argv[1:])
