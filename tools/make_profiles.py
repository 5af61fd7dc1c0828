#!/usr/bin/env python
"""Turn one round's ncu outputs (gpurun_out/) into the tracked summaries under profiles/.

usage: tools/make_profiles.py TAG [launches.csv] [full.ncu-rep ...]
  - launches csv (`ncu --metrics gpu__time_duration.sum --clock-control none --csv`): per-launch list
    (copied verbatim) and a per-kernel table (count, mean / min / max us) with each decode kernel's share
    of the decode step (classify + compact_alloc + quant_write);
  - each --set full capture: headline metrics per kernel plus dram__bytes_read/write.sum (the `traffic`
    figure bench.py reports) written to profiles/TAG_<capture>.md and profiles/traffic.json.
"""
import csv
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

DETAILS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L2 Hit Rate",
           "L1/TEX Hit Rate", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
           "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Issue Slots Busy",
           "Grid Size", "Block Size", "Executed Instructions")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active")


def _csv_rows(text):
    rows = list(csv.reader(text.splitlines()))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    return rows[i], rows[i + 1:]


def short(name):
    return name.split("(")[0].replace("void ", "")


def launches(tag, path):
    h, rows = _csv_rows(open(path).read())
    per = {}
    order = []
    for r in rows:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d.get("Metric Unit", "nsecond")
        v = float(d["Metric Value"].replace(",", ""))
        us = v / 1000.0 if unit.startswith("n") else (v * 1000.0 if unit.startswith("m") else v)
        k = short(d["Kernel Name"])
        per.setdefault(k, []).append(us)
        order.append((int(d["ID"]), k, us))
    with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
        f.write("id,kernel,us\n")
        for i, k, us in order:
            f.write(f"{i},{k},{us:.3f}\n")
    # the memory manager's decode-step kernels (NEXT-2's attention is model compute, reported on its own)
    dec = [(k, us) for i, k, us in order
           if any(x in k for x in ("classify_decode", "compact_alloc", "quant_decode", "recycle_kernel"))]
    dper = {}
    for k, us in dec:
        dper.setdefault(k, []).append(us)
    # per-step cost: a kernel's total over the decode phase / the number of steps (one classify per step), so the
    # recycle kernel, which runs only in the steps that free a request, counts at its amortised cost
    nsteps = max((len(v) for k, v in dper.items() if "classify_decode" in k), default=0) or 1
    cost = {k: sum(v) / nsteps for k, v in dper.items()}
    step = sum(cost.values())
    lines = [f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)", "",
             "Per-launch times are cold-cache and serialised (ncu replays each launch alone); the SHARE of each",
             "kernel in the decode step is what bench.py's live CUDA-event timing must agree with.", "",
             "| kernel | launches | mean us | min us | max us | share of decode step |",
             "|---|---|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        share = ""
        if k in dper:
            share = f"{100 * cost[k] / step:.1f}%"
        lines.append(f"| {k} | {len(v)} | {statistics.mean(v):.2f} | {min(v):.2f} | {max(v):.2f} | {share} |")
    lines += ["", f"Decode step ({len(dec)} decode-phase launches over {nsteps} steps, per-step total): {step:.2f} us", ""]
    return "\n".join(lines)


def capture(tag, path):
    name = os.path.splitext(os.path.basename(path))[0]
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    h, rows = _csv_rows(det)
    kern = {}
    for r in rows:
        d = dict(zip(h, r))
        key = (int(d["ID"]), short(d["Kernel Name"]))
        if d["Metric Name"] in DETAILS:
            kern.setdefault(key, {})[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh = rr[0]
    units = dict(zip(hh, rr[1]))
    rawk = {}
    for r in rr[2:]:
        d = dict(zip(hh, r))
        key = (int(d["ID"]), short(d["Kernel Name"]))
        rawk[key] = {m: (d.get(m), units.get(m)) for m in RAW}
    out = [f"# {tag}: `ncu --set full --import-source on --clock-control none` capture `{name}`", ""]
    traffic = {}
    for key in sorted(kern):
        out.append(f"## [{key[0]}] {key[1]}")
        out.append("")
        for m in DETAILS:
            if m in kern[key]:
                out.append(f"- {m}: {kern[key][m]}")
        for m, (v, u) in rawk.get(key, {}).items():
            if v is not None:
                out.append(f"- `{m}`: {v} {u or ''}")
        rb = rawk.get(key, {}).get("dram__bytes_read.sum", (None, None))
        wb = rawk.get(key, {}).get("dram__bytes_write.sum", (None, None))
        if rb[0] and wb[0]:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tb = float(rb[0].replace(",", "")) * scale.get(rb[1], 1) + float(wb[0].replace(",", "")) * scale.get(wb[1], 1)
            traffic.setdefault(key[1], tb)
            out.append(f"- DRAM traffic (read + write): {tb / 1e6:.3f} MB per launch")
        out.append("")
    with open(os.path.join(PROF, f"{tag}_{name}.md"), "w") as f:
        f.write("\n".join(out))
    return traffic


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    tj = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            md = launches(tag, a)
            with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
                f.write(md)
            print(md)
        elif a.endswith(".ncu-rep"):
            t = capture(tag, a)
            for k, v in t.items():
                traffic[k] = {"bytes_per_launch": v, "source": f"profiles/{tag}_{os.path.splitext(os.path.basename(a))[0]}.md"}
            print(a, t)
    with open(tj, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
