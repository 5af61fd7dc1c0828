#!/usr/bin/env python
"""Dynamic SASS opcode mix of one kernel from an .ncu-rep (source page, sass view): executed warp instructions
per opcode and the stall samples on them.  usage: tools/sass_dyn.py REP KERNEL_REGEX [top]"""
import collections
import csv
import subprocess
import sys


def main(path, kre, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    ie, ns, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    ins, smp = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        op = r[src].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1]
        o = o.split(".")[0]
        try:
            ins[o] += int(r[ie])
            smp[o] += int(r[ns])
        except ValueError:
            pass
    tot, ts = sum(ins.values()), sum(smp.values())
    print(f"total {tot} warp instructions, {ts} stall samples")
    for o, n in ins.most_common(top):
        print(f"{o:10s} {n:12d} {100 * n / tot:5.1f}%   samples {100 * smp[o] / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
