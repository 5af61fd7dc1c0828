#!/usr/bin/env python
"""Debug probe for dkv_attend_tc: tiny pools, the error structure of the outputs / probabilities against Eq. 1 in
float64 (per feature, per head, stored vs window tokens)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests import eq1  # noqa: E402
from tests import harness as H  # noqa: E402
from tests.gpu_backend import GpuBackend  # noqa: E402

np.set_printoptions(precision=4, suppress=True, linewidth=200)
for G, d, W, lens in ((1, 128, 64, [520, 70, 300]), (4, 128, 64, [520, 70, 300]), (4, 128, 64, [16, 40, 200])):
    scn = H.TINY.replace(R=3, Ly=1, H=1, d=d, M=700, W=W, P=6000, seed=21, q_per_kv=G, alpha_h=1.0, alpha_l=0.02)
    g = GpuBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([g], inp, life, list(range(len(lens))), lens)
    q = np.random.default_rng(G).normal(0, 1, size=(scn.U, G, d)).astype(np.float16)
    snap = g.snapshot()
    _, og, pg = g.attend_tc(q, want_out=True, want_probs=True)
    for u in range(scn.U):
        k, v, pos = eq1.unit_tokens64(snap["pages"], snap["table"][u], snap["n_h"][u], snap["n_l"][u],
                                      snap["seq_len"][u], snap["win_k"][u], snap["win_v"][u], g.geom, g.L, W, d)
        ref, rp = eq1.attend64(q[u], k, v)
        err = np.abs(og[u] - ref)
        n = len(pos)
        perr = np.abs(pg[u][:n] - rp)
        nh, nl = int(snap["n_h"][u]), int(snap["n_l"][u])
        print(f"G={G} u={u} n_h={nh} n_l={nl} T={n} out max err {err.max():.3e} (|ref| max {np.abs(ref).max():.3f}) "
              f"probs max err: high {perr[:nh].max() if nh else 0:.2e} low {perr[nh:nh+nl].max() if nl else 0:.2e} "
              f"win {perr[nh+nl:].max():.2e}  sum p gpu {pg[u][:n].sum():.4f} ref {rp.sum():.4f}")
        if err.max() > 1e-3:
            print("  err by feature (max over heads):", err.max(0)[:32])
            print("  got[0,:8]", og[u][0][:8], "ref", ref[0][:8])
            # ratio test: got vs ref as a linear fit
            a = np.polyfit(ref.ravel(), og[u].ravel(), 1)
            print("  fit got = a*ref + b:", a)
