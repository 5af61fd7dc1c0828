#!/usr/bin/env python
"""Tensor-core attention timing at few-unit, long-context shapes (where the split-sequence form applies): mean ms of
dkv_attend_tc over 5 calls (CUDA events), per shape.  Run it on builds with -DDKV_TC_SPLIT=0 / 1 to compare."""
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests import harness as H  # noqa: E402
from tests.gpu_backend import GpuBackend  # noqa: E402

for name, kw, lens in (("1 req x 2 heads, 30k", dict(R=1, Ly=1, H=2, M=33792, P=4000, q_per_kv=8, alpha_l=0.0,
                                                      mix=(0.4, 0.6, 0.0)), [30000]),
                       ("4 req x 8 heads, 16k", dict(R=4, Ly=1, H=8, M=17408, P=40000, q_per_kv=4), [16000] * 4),
                       ("16 req x 8 heads, 8k", dict(R=16, Ly=1, H=8, M=9216, P=90000, q_per_kv=4), [8000] * 16),
                       ("32 req x 8 heads, 8k", dict(R=32, Ly=1, H=8, M=9216, P=180000, q_per_kv=4), [8000] * 32)):
    scn = H.TINY.replace(d=128, W=64, seed=13, alpha_h=1.0, **kw)
    g = GpuBackend(scn)
    H.admit([g], H.Inputs(scn), H.Lifecycle(scn), list(range(len(lens))), lens)
    G = scn.q_per_kv
    q = torch.from_numpy(np.random.default_rng(1).normal(size=(scn.U, G, 128)).astype(np.float16).view(np.int16)).cuda()
    out = torch.empty((scn.U, G, 128), dtype=torch.float32, device="cuda")
    ts = []
    for i in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.pool.attend_tc(q, out)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    print(f"{name}: {statistics.mean(ts):.3f} ms ({scn.U} units)")
    del g
