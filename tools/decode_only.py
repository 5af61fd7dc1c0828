#!/usr/bin/env python
"""configs[1] decode steps only (prefill once, then `--steps` eager decode steps with the bench's drift, churn-free)
— a short host program for targeted ncu captures of the decode kernels:
    ncu --set full -k regex:quant_decode -s 8 -c 1 -o out python tools/decode_only.py --steps 12
Optional --attend {exact,tc}: one attention call after each decode step (NEXT-2)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2412_03131_b200 import Pool  # noqa: E402
from paper_2412_03131_b200 import dkv as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--attend", default="", choices=["", "exact", "tc"])
    a = ap.parse_args()
    c = bench.CONFIGS["llama3_8b"]
    dev = torch.device("cuda", 0)
    wl = bench.Workload(c, 0, 1, dev)
    cfg = D.make_config(wl.R, c["Ly"], wl.Hl, c["d"], c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"],
                        alpha_h=c["alpha_h"], alpha_l=c["alpha_l"], q_per_kv=c["G"])
    pool = Pool(cfg, device=dev)
    geom = pool.geom()
    T = c["prompt"]
    sig, kk, vv = wl.prefill_inputs(T)
    pool.classify_prefill(list(range(wl.R)), [T] * wl.R, sig)
    pool.compact_alloc(None)
    pool.quant_write_prefill(kk.view(torch.int16), vv.view(torch.int16), sig)
    del sig, kk, vv
    import numpy as np
    seq = np.full(wl.R, T, np.int64)
    active = np.ones(wl.R, bool)
    dec = pool.new_decisions()
    q = torch.empty((wl.U, c["G"], c["d"]), dtype=torch.float16, device=dev)
    out = torch.empty((wl.U, c["G"], c["d"]), dtype=torch.float32, device=dev)
    for s in range(a.steps):
        v = pool.views()
        synth.apply_drift(c["seed"], s, wl.shape, v["pages"], v["table"], v["n_h"], v["n_l"],
                          {k_: (geom[k_]["C"], geom[k_]["off_score"], geom[k_]["off_pos"]) for k_ in (1, 2)}, pool.L)
        cand, nk, nv = wl.decode_inputs(seq, active)
        pool.classify_decode(cand, dec)
        pool.compact_alloc(dec)
        pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), cand)
        seq += 1
        if a.attend:
            q.normal_()
            (pool.attend if a.attend == "exact" else pool.attend_tc)(q.view(torch.int16), out)
    torch.cuda.synchronize()
    st, _ = pool.query()
    assert st == 0, st
    print("ok", a.steps)


if __name__ == "__main__":
    main()
