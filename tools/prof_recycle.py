"""Set up the Llama-3-8B-shaped pool (bench.py configs[1]), free `--nfree` requests and run one decode step
whose dkv_compact_alloc recycles them, inside an NVTX range "recycle" (for ncu --nvtx-include)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_03131_b200 import Pool  # noqa: E402
from paper_2412_03131_b200 import dkv as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nfree", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
c = bench.CONFIGS["llama3_8b"]
dev = torch.device("cuda", 0)
wl = bench.Workload(c, 0, 1, dev)
T = c["prompt"]
cfg = D.make_config(wl.R, c["Ly"], wl.Hl, c["d"], c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"], alpha_h=c["alpha_h"],
                    alpha_l=c["alpha_l"])
pool = Pool(cfg, device=dev)
sig, kk, vv = wl.prefill_inputs(T)
reqs = list(range(wl.R))
dec = pool.new_decisions()
seq = np.full(wl.R, T, np.int64)
act = np.ones(wl.R, bool)
pool.classify_prefill(reqs, [T] * wl.R, sig)
pool.compact_alloc(None)
pool.quant_write_prefill(kk.view(torch.int16), vv.view(torch.int16), sig)
times = []
for rep in range(a.reps):
    fr = [(rep * 7 + i * 13) % wl.R for i in range(a.nfree)]
    pool.free(fr)
    act[fr] = False
    cand, nk, nv = wl.decode_inputs(seq, act)
    pool.classify_decode(cand, dec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("recycle")
    e0.record()
    pool.compact_alloc(dec)
    e1.record()
    torch.cuda.nvtx.range_pop()
    pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), cand)
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) * 1e3)
    seq[act] += 1
    pool.classify_prefill(fr, [T] * len(fr), sig[fr])
    pool.compact_alloc(None)
    pool.quant_write_prefill(kk[fr].view(torch.int16), vv[fr].view(torch.int16), sig[fr])
    seq[fr] = T
    act[fr] = True
st, stats = pool.query()
print("recycle compact_alloc us:", [round(t, 1) for t in times], "status", st, "last_freed", stats.last_freed)
