#!/usr/bin/env python
"""configs[1] eager decode steps (bench.py's drift, L2 flush, CUDA events): mean / p50 us of classify,
compact_alloc and quant_write over 20 steps — a fast A/B probe for decode-kernel build variants."""
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2412_03131_b200 import Pool  # noqa: E402
from paper_2412_03131_b200 import dkv as D  # noqa: E402

c = bench.CONFIGS["llama3_8b"]
dev = torch.device("cuda", 0)
wl = bench.Workload(c, 0, 1, dev)
cfg = D.make_config(wl.R, c["Ly"], wl.Hl, c["d"], c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"], alpha_h=c["alpha_h"],
                    alpha_l=c["alpha_l"], q_per_kv=c["G"])
pool = Pool(cfg, device=dev)
geom = pool.geom()
T = c["prompt"]
sig, kk, vv = wl.prefill_inputs(T)
pool.classify_prefill(list(range(wl.R)), [T] * wl.R, sig)
pool.compact_alloc(None)
pool.quant_write_prefill(kk.view(torch.int16), vv.view(torch.int16), sig)
del sig, kk, vv
seq = np.full(wl.R, T, np.int64)
active = np.ones(wl.R, bool)
dec = pool.new_decisions()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {"classify": [], "compact": [], "quant": []}
for s in range(25):
    v = pool.views()
    synth.apply_drift(c["seed"], s, wl.shape, v["pages"], v["table"], v["n_h"], v["n_l"],
                      {k_: (geom[k_]["C"], geom[k_]["off_score"], geom[k_]["off_pos"]) for k_ in (1, 2)}, pool.L)
    cand, nk, nv = wl.decode_inputs(seq, active)
    flush.zero_()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda._sleep(200_000)
    e[0].record()
    pool.classify_decode(cand, dec)
    e[1].record()
    pool.compact_alloc(dec)
    e[2].record()
    pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), cand)
    e[3].record()
    torch.cuda.synchronize()
    seq += 1
    if s >= 5:
        res["classify"].append(e[0].elapsed_time(e[1]) * 1e3)
        res["compact"].append(e[1].elapsed_time(e[2]) * 1e3)
        res["quant"].append(e[2].elapsed_time(e[3]) * 1e3)
st, _ = pool.query()
assert st == 0
print(" ".join(f"{k}={statistics.mean(v):.2f}/{np.percentile(v, 50):.2f}" for k, v in res.items()))
