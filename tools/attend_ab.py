#!/usr/bin/env python
"""configs[1] NEXT-2 attention timing probe: prefill, 3 decode steps, then exact and tensor-core attention
(CUDA events, L2 flushed), mean ms of each over 5 calls."""
import os
import statistics
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
q = torch.randn((wl.U, c["G"], c["d"]), device=dev).to(torch.float16)
out = torch.empty((wl.U, c["G"], c["d"]), dtype=torch.float32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
impls = (("exact", pool.attend), ("tc", pool.attend_tc))
if os.environ.get("ONLY"):                                     # e.g. ONLY=tc under ncu
    impls = tuple(x for x in impls if x[0] == os.environ["ONLY"])
for name, fn in impls:
    ts = []
    for i in range(6):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(q.view(torch.int16), out)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    res[name] = statistics.mean(ts)
st, _ = pool.query()
assert st == 0
print(" ".join(f"{k}={v:.3f}ms" for k, v in res.items()))
