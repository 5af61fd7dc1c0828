#!/usr/bin/env python
"""Top SASS lines by warp-stall samples for one kernel of an .ncu-rep, with their dominant stall reasons."""
import csv
import subprocess
import sys


def main(path, kernel_regex, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kernel_regex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    # the file may contain several kernels; take the first block
    start = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[start]
    data = []
    for r in rows[start + 1:]:
        if not r or r[0] == "Kernel Name" or r[0] == "Address":
            break
        if len(r) == len(h):
            data.append(r)
    smp = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(r[smp] or 0) for r in data)
    print("samples", tot, "instructions", len(data))
    for r in sorted(data, key=lambda r: -int(r[smp] or 0))[:top]:
        st = sorted(((int(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:3]
        print(f"{int(r[smp]):7d} {100 * int(r[smp]) / max(tot, 1):5.1f}%  {r[src][:70]:70s} {[(n, v) for v, n in st if v]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
