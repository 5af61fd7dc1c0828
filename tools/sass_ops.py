#!/usr/bin/env python
"""Static SASS opcode histogram of the kernels in an object / library whose mangled name matches a pattern
(cuobjdump -sass): a quick check of what a source change did to the instruction mix, before GPU time."""
import collections
import re
import subprocess
import sys


def main(path, pat, top=25):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, hist = None, {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1) if re.search(pat, m.group(1)) else None
            if cur:
                hist[cur] = collections.Counter()
            continue
        if cur:
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                hist[cur][m.group(2).split(".")[0]] += 1
    for f, h in hist.items():
        print(f, sum(h.values()))
        print("   ", ", ".join(f"{k} {v}" for k, v in h.most_common(top)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
