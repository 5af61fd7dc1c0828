#!/usr/bin/env python
"""Measurements at BASELINE.json's other workload shapes, one GPU's shard each (bench.py's headline line is
configs[1]; the driver runs only that).  One JSON line per config:

  qwen32b_thinking : configs[2] — Qwen-32B-style thinking workload: 32 requests x 64 layers x 8 KV heads,
                     GQA group 5, contexts grown to 16k of a 33k budget, no pruning (alpha_l = 0), churn (one
                     request finishes and a new 16k one is admitted every 4 steps); attention runs the
                     long-context form (logits in HBM slots)
  llama70b_shard8  : configs[3] — Llama-3-70B, batch 256 x 8k, 80 layers, the 8 KV heads partitioned 8-way:
                     this GPU's pool holds one head (20480 units), GQA group 8
  frag_shard8      : configs[4] — fragmentation stress: 1024 requests of random lengths (256..4096), random
                     finish order, admission keeps the pool near 90 % occupancy, 400 steps of alloc / free;
                     one head of 8 per GPU (32768 units)

Per config: bulk quant-write GB/s over the admissions, then decode steps timed with CUDA events on the pool's
stream (L2 flushed before each): classify (scan) / compact_alloc / quant_write µs, and the NEXT-2 step
(attend + classify from the section minima).  Inputs are seeded synthetic (synth/), as in bench.py.
usage: python tools/bench_configs.py [name ...]
"""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2412_03131_b200 import Pool  # noqa: E402
from paper_2412_03131_b200 import dkv as D  # noqa: E402

# R is per shard-group member: bench.Workload multiplies it by `world` (here the shard count) and keeps H/world
# heads, so world = 8 gives the 8-way head partition of one GPU with the full request batch
SHAPES = {
    # configs[1] (bench.py's headline shape) through this harness, with the paper's prompt workflow (NEXT-1,
    # conservative allocation + reclaim) and with per-(layer, head) thresholds (NEXT-4)
    "llama3_8b": dict(R=64, Ly=32, H=8, world=1, d=128, prompt=4096, M=8192, W=64, Ch=16, Cl=32, P=1 << 22,
                      alpha_h=1.0, alpha_l=0.02, mix=(0.35, 0.45, 0.20), seed=2, G=4, steps=12, churn_every=4,
                      group=64),
    "llama3_8b_workflow1": dict(R=64, Ly=32, H=8, world=1, d=128, prompt=4096, M=8192, W=64, Ch=16, Cl=32,
                                P=1 << 22, alpha_h=1.0, alpha_l=0.02, mix=(0.35, 0.45, 0.20), seed=2, G=4, steps=12,
                                churn_every=4, group=64, workflow=1),
    "llama3_8b_head_thresholds": dict(R=64, Ly=32, H=8, world=1, d=128, prompt=4096, M=8192, W=64, Ch=16, Cl=32,
                                      P=1 << 22, alpha_h=1.0, alpha_l=0.02, mix=(0.35, 0.45, 0.20), seed=2, G=4,
                                      steps=12, churn_every=4, group=64, head_alpha=True),
    "qwen32b_thinking": dict(R=32, Ly=64, H=8, world=1, d=128, prompt=16384, M=33792, W=64, Ch=16, Cl=32,
                             P=14 << 20, alpha_h=3.0, alpha_l=0.0, mix=(0.4, 0.6, 0.0), seed=3, G=5, steps=12,
                             churn_every=4, group=1),
    # SURVEY §8(d) / P:703: alpha (1, 0) for Llama-3-70B, no pruning, mix .25 / .75 / 0
    "llama70b_shard8": dict(R=32, Ly=80, H=8, world=8, d=128, prompt=8192, M=9216, W=64, Ch=16, Cl=32,
                            P=7 << 20, alpha_h=1.0, alpha_l=0.0, mix=(0.25, 0.75, 0.0), seed=4, G=8, steps=12,
                            churn_every=4, group=16),
    # NEXT-4 three-level tier FP16-K8V4-K4V2 (readings Q38-Q44) on configs[1]'s shape; no attention (Q44)
    # (about 42 % of the stored prompt tokens reach alpha_t / n here, at 4 tokens per page: 12 Mi pages)
    "llama3_8b_top_tier": dict(R=64, Ly=32, H=8, world=1, d=128, prompt=4096, M=8192, W=64, Ch=16, Cl=32,
                               P=12 << 20, alpha_h=1.0, alpha_l=0.02, mix=(0.35, 0.45, 0.20), seed=2, G=4, steps=12,
                               churn_every=4, group=64, top_tier=1, alpha_t=2.0, Ct=4),
    "frag_shard8": dict(R=128, Ly=32, H=8, world=8, d=128, prompt=(256, 4096), M=4608, W=64, Ch=16, Cl=32,
                        P=2_900_000, alpha_h=1.0, alpha_l=0.02, mix=(0.35, 0.45, 0.20), seed=5, G=4, steps=400,
                        churn_every=1, group=64, occupancy=0.90),
}


def ev():
    return torch.cuda.Event(enable_timing=True)


def run(name):
    c = dict(SHAPES[name])
    dev = torch.device("cuda", 0)
    wl = bench.Workload(c, 0, c["world"], dev)
    rng = np.random.default_rng(c["seed"])
    ragged = isinstance(c["prompt"], tuple)
    Tmax = c["prompt"][1] if ragged else c["prompt"]
    cfg = D.make_config(wl.R, c["Ly"], wl.Hl, c["d"], c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"],
                        alpha_h=c["alpha_h"], alpha_l=c["alpha_l"], q_per_kv=c["G"],
                        prefill_workflow=c.get("workflow", 0), top_tier=c.get("top_tier", 0),
                        alpha_t=c.get("alpha_t", 0.0), page_tokens_top=c.get("Ct", 4))
    pool = Pool(cfg, device=dev)
    if c.get("head_alpha"):                                      # per-(layer, head) pairs around the pool-wide one
        hr = np.random.default_rng(c["seed"] + 99)
        f = hr.uniform(0.5, 2.0, size=c["Ly"] * wl.Hl)
        assert pool.set_head_thresholds((c["alpha_h"] * f).astype(np.float32).tolist(),
                                        (c["alpha_l"] * f).astype(np.float32).tolist()) == 0
    geom = pool.geom()
    dec = pool.new_decisions()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    seq = np.zeros(wl.R, np.int64)
    active = np.zeros(wl.R, bool)
    bulk = {"ms": 0.0, "bytes": 0}
    plan_us = []                                                 # classify(PREFILL) + compact_alloc per admission

    def admit(reqs):
        lens = [int(rng.integers(c["prompt"][0], c["prompt"][1] + 1)) if ragged else Tmax for _ in reqs]
        T = max(lens)
        sig = torch.empty((len(reqs), wl.LyH, T), dtype=torch.float32, device=dev)
        k = torch.empty((len(reqs), wl.LyH, T, c["d"]), dtype=torch.float16, device=dev)
        v = torch.empty_like(k)
        for i, r in enumerate(reqs):
            ln = torch.full((wl.LyH,), lens[i], dtype=torch.int64, device=dev)
            sig[i] = synth.prefill_sig(c["seed"], wl.ug[r], T, c["alpha_h"], c["alpha_l"], wl.mix_h[r],
                                       wl.mix_l[r], lens=ln)
            for j0 in range(0, wl.LyH, 64):
                g = wl.ug[r, j0:j0 + 64]
                k[i, j0:j0 + 64] = synth.kv_values(c["seed"], synth.S_KEY, g, 0, T, c["d"])
                v[i, j0:j0 + 64] = synth.kv_values(c["seed"], synth.S_VAL, g, 0, T, c["d"])
        nh0, nl0 = pool.views()["n_h"].sum().item(), pool.views()["n_l"].sum().item()
        torch.cuda.synchronize()
        p0, p1 = ev(), ev()
        torch.cuda._sleep(200_000)                               # host submission ahead of the timed region
        p0.record()
        pool.classify_prefill(list(reqs), lens, sig)
        pool.compact_alloc(None)
        p1.record()
        torch.cuda.synchronize()
        plan_us.append(p0.elapsed_time(p1) * 1e3)
        e0, e1 = ev(), ev()
        torch.cuda._sleep(200_000)
        e0.record()
        pool.quant_write_prefill(k.view(torch.int16), v.view(torch.int16), sig)
        e1.record()
        torch.cuda.synchronize()
        st, _ = pool.query()
        assert st == 0, f"status {st} after admission"
        vv = pool.views()
        nh = vv["n_h"].sum().item() - nh0
        nl = vv["n_l"].sum().item() - nl0
        units, kept = len(reqs) * wl.LyH, sum(max(t - c["W"], 0) for t in lens) * wl.LyH
        rd = 4 * c["d"] + 4
        hb = rd + geom[1]["k_row"] + geom[1]["v_row"] + 16
        lb = rd + geom[2]["k_row"] + geom[2]["v_row"] + 16
        nw = sum(min(c["W"], t) for t in lens) * wl.LyH
        bulk["ms"] += e0.elapsed_time(e1)
        bulk["bytes"] += nh * hb + nl * lb + (kept - nh - nl) * 4 + nw * 4 * c["d"]
        for i, r in enumerate(reqs):
            seq[r], active[r] = lens[i], True
        del sig, k, v
        return units

    def occupancy():
        _, stats = pool.query()
        return 1.0 - stats.free_pages / c["P"]

    # ---- admissions
    t0 = time.time()
    target = c.get("occupancy")
    order = list(range(wl.R))
    for i in range(0, wl.R, c["group"]):
        if target is not None and occupancy() > target:
            break
        admit(order[i:i + c["group"]])
    admit_s = time.time() - t0

    # ---- decode steps (significance from the synthetic input), then NEXT-2 steps (from the attention)
    res = {k_: [] for k_ in ("classify", "compact_alloc", "quant_write", "attend", "attend_tc", "classify_fused",
                             "occ")}
    freed = admitted = 0
    qbuf = torch.empty((wl.U, c["G"], c["d"]), dtype=torch.float16, device=dev)
    obuf = torch.empty((wl.U, c["G"], c["d"]), dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(c["seed"])
    for s in range(c["steps"]):
        next2 = s >= c["steps"] // 2 and not c.get("top_tier")     # Q44: no attention with the FP16 tier
        tc_ok = c["Ch"] == 16 and c["Cl"] == 32                  # attend_tc's specialisation (K8V4 x16, K4V2 x32)
        if s % c["churn_every"] == c["churn_every"] - 1:
            live = np.nonzero(active)[0]
            if len(live):
                r = int(rng.choice(live))                       # random finish order
                pool.free([r])
                active[r] = False
                freed += 1
        cand, nk, nv = wl.decode_inputs(seq, active)
        if next2:
            qbuf.normal_(generator=gen)
        if next2 and tc_ok:                                      # the tensor-core attention on the same state,
            flush.zero_()                                         # before the exact one (whose minima drive the step)
            torch.cuda.synchronize()
            t0e, t1e = ev(), ev()
            torch.cuda._sleep(200_000)
            t0e.record()
            pool.attend_tc(qbuf.view(torch.int16), obuf)
            t1e.record()
            torch.cuda.synchronize()
            res["attend_tc"].append(t0e.elapsed_time(t1e) * 1e3)
        flush.zero_()
        torch.cuda.synchronize()
        e = [ev() for _ in range(5)]
        torch.cuda._sleep(200_000)
        e[0].record()
        if next2:
            pool.attend(qbuf.view(torch.int16), obuf)
        e[1].record()
        pool.classify_decode(None if next2 else cand, dec)
        e[2].record()
        pool.compact_alloc(dec)
        e[3].record()
        pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), None if next2 else cand)
        e[4].record()
        torch.cuda.synchronize()
        seq[active] += 1
        if next2:
            res["attend"].append(e[0].elapsed_time(e[1]) * 1e3)
            res["classify_fused"].append(e[1].elapsed_time(e[2]) * 1e3)
        else:
            res["classify"].append(e[1].elapsed_time(e[2]) * 1e3)
        res["compact_alloc"].append(e[2].elapsed_time(e[3]) * 1e3)
        res["quant_write"].append(e[3].elapsed_time(e[4]) * 1e3)
        st, _ = pool.query()
        assert st == 0, f"status {st} at step {s}"
        # re-admit into free slots while the pool stays below the target occupancy (or keep the batch full)
        idle = np.nonzero(~active)[0]
        if len(idle) and (target is None or occupancy() < target):
            admit([int(idle[0])])
            admitted += 1
        res["occ"].append(occupancy())
    # pool-wide invariant at the end: page ownership is a permutation of 0..P-1
    v = pool.views()
    ctrl = v["ctrl"].cpu().numpy()
    start, free = int(ctrl[0]), int(ctrl[1])
    ids = torch.cat([v["ring"][(start + torch.arange(free, device=dev)) % c["P"]], v["table"][v["table"] >= 0],
                     v["ttable"][v["ttable"] >= 0]])
    assert ids.numel() == c["P"] and torch.equal(ids.sort().values, torch.arange(c["P"], device=dev, dtype=ids.dtype))

    def m(k_):
        return round(statistics.mean(res[k_]), 2) if res[k_] else None

    return {"config": name, "units": wl.U, "shard": f"{wl.Hl} of {c['H']} KV heads", "requests": wl.R,
            "q_per_kv": c["G"], "pages": c["P"],
            "bulk_quant_write": {"gbs": round(bulk["bytes"] / (bulk["ms"] * 1e-3) / 1e9, 1),
                                 "algorithmic_bytes": int(bulk["bytes"]), "ms_total": round(bulk["ms"], 2)},
            "prefill_plan_us": {"first_admission": round(plan_us[0], 1),
                                "single_request_mean": round(statistics.mean(plan_us[1:]), 1) if len(plan_us) > 1
                                else None},
            "prefill_workflow": c.get("workflow", 0), "per_head_thresholds": bool(c.get("head_alpha")),
            "decode_us": {"classify_scan": m("classify"), "compact_alloc": m("compact_alloc"),
                          "quant_write": m("quant_write"), "classify_fused": m("classify_fused"),
                          "compact_alloc_p99": round(float(np.percentile(res["compact_alloc"], 99)), 2)},
            "attend_ms": round(m("attend") / 1e3, 3) if res["attend"] else None,
            "attend_tc_ms": round(m("attend_tc") / 1e3, 3) if res["attend_tc"] else None,
            "steps": c["steps"], "frees": freed, "admissions_during_decode": admitted,
            "occupancy": {"min": round(min(res["occ"]), 3), "max": round(max(res["occ"]), 3)},
            "mean_context": int(seq[active].mean()) if active.any() else 0, "admit_s": round(admit_s, 1),
            "data": "synthetic (synth/, seeded)", "l2": "flushed before every timed step"}


def warm_up(seconds=3.0):
    """Bring the GPU out of idle clocks before the first config is timed (copies over 2 GiB buffers)."""
    a = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    t0 = time.time()
    while time.time() - t0 < seconds:
        b.copy_(a)
        torch.cuda.synchronize()
    del a, b
    torch.cuda.empty_cache()


if __name__ == "__main__":
    names = sys.argv[1:] or list(SHAPES)
    warm_up()
    # throwaway pass of the first config: the first pool of the process measured 20-70 % slow (first touch of
    # its pages, module load), profiles/r1f_configs.jsonl
    run(names[0])
    torch.cuda.empty_cache()
    for n in names:
        print(json.dumps(run(n)), flush=True)
        torch.cuda.empty_cache()
