#!/usr/bin/env python
"""compact_alloc phase timing from a -DDKV_CA_TRACE=1 build: configs[1] decode steps (no frees), after each
dkv_compact_alloc the last tile's globaltimer marks (entry, after the loads, after the warp scans, after the
look-back, after the grant, exit) from rec[0..11]; prints the mean phase durations in ns."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2412_03131_b200 import Pool  # noqa: E402
from paper_2412_03131_b200 import dkv as D  # noqa: E402

c = bench.CONFIGS["llama3_8b"]
dev = torch.device("cuda", 0)
wl = bench.Workload(c, 0, 1, dev)
cfg = D.make_config(wl.R, c["Ly"], wl.Hl, c["d"], c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"], alpha_h=c["alpha_h"],
                    alpha_l=c["alpha_l"], q_per_kv=c["G"])
pool = Pool(cfg, device=dev)
T = c["prompt"]
sig, kk, vv = wl.prefill_inputs(T)
pool.classify_prefill(list(range(wl.R)), [T] * wl.R, sig)
pool.compact_alloc(None)
pool.quant_write_prefill(kk.view(torch.int16), vv.view(torch.int16), sig)
del sig, kk, vv
seq = np.full(wl.R, T, np.int64)
act = np.ones(wl.R, bool)
dec = pool.new_decisions()
off = int(pool.layout.off_rec)
marks = []
for s in range(12):
    cand, nk, nv = wl.decode_inputs(seq, act)
    pool.classify_decode(cand, dec)
    torch.cuda.synchronize()
    pool.compact_alloc(dec)
    torch.cuda.synchronize()
    m = pool.arena[off:off + 48].view(torch.int64).cpu().numpy().copy()
    pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), cand)
    seq += 1
    if s >= 2:
        marks.append(np.diff(m))
d = np.mean(marks, axis=0)
names = ["loads+barrier1", "warp scans+barrier2", "tile prefix+barrier3", "recycle block+grant", "transitions+pointers"]
for n, v in zip(names, d):
    print(f"{n:24s} {v:8.0f} ns")
print(f"{'entry->exit (last tile)':24s} {sum(d):8.0f} ns")
