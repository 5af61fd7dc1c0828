#!/usr/bin/env python
"""Executed warp instructions and stall samples per CUDA source line of one kernel of an .ncu-rep
(the cuda,sass source page): where a kernel's instruction budget goes."""
import csv
import subprocess
import sys


def main(path, kernel_regex, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kernel_regex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg, fname, h, tot = [], "", None, 0
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        elif r and r[0] == "Line No":
            h = r
        elif h and r and r[0] not in ("", "Function Name", "Kernel Name", "File Name"):
            d = dict(zip(h[:3], r[:3]))
            try:
                ins = int(r[h.index("Instructions Executed")])
                smp = int(r[h.index("# Samples")])
            except (ValueError, IndexError):
                continue
            tot += ins
            agg.append((ins, smp, f"{fname}:{r[0]}", r[1][:110]))
    agg.sort(reverse=True)
    print(f"total warp instructions {tot}")
    for ins, smp, loc, src in agg[:top]:
        print(f"{ins:>12} {100 * ins / max(tot, 1):5.1f}% {smp:>7}  {loc:<22} {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
