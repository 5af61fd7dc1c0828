#!/usr/bin/env python
"""Summarise an .ncu-rep (details page) per kernel: key throughput / occupancy / stall metrics."""
import csv
import subprocess
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size", "Mem Busy", "Max Bandwidth")


def main(path, raw_metrics=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    seen = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"][:48])
        if d["Metric Name"] in WANT:
            seen.setdefault(key, []).append(f"{d['Metric Name']}={d['Metric Value']}{d['Metric Unit']}")
    for (i, k), v in seen.items():
        print(f"[{i}] {k}")
        for x in v:
            print("     ", x)
    if raw_metrics:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h = rows[0]
        for r in rows[2:]:
            d = dict(zip(h, r))
            print(d.get("Kernel Name", "")[:48], {m: d.get(m) for m in raw_metrics})


if __name__ == "__main__":
    main(sys.argv[1], tuple(sys.argv[2:]))
