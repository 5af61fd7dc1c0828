#!/usr/bin/env python
"""bench.py — DiffKV on-GPU KV memory manager on B200 (arXiv 2412.03131), BASELINE.json's metric:
"µs per decode-step compact+alloc (64 req×32L×8H); quant-write GB/s vs HBM peak, 1/2/4/8 GPU".

Workload (BASELINE configs[1]): Llama-3-8B KV shape — 64 requests x 32 layers x 8 KV heads
per GPU (16,384 units), head_dim 128, 4096-token prompts, max 8192 tokens, W = 64, K8V4 (16-token pages)
/ K4V2 (32-token pages), 2^22 pages (15 GB) per GPU, alpha_h = 1, alpha_l = 0.02, seeded synthetic
significance / K / V (synth/).  At N GPUs the global batch is 64*N requests and the 8 KV heads are
sharded N-way (one independent pool per GPU): per-GPU work is constant ("weak" scaling).

Phases (each bracketed by barrier + synchronize, every kernel timed with CUDA events on its stream):
  bulk   : K rounds of dkv_quant_write(PREFILL) of the whole batch (the HBM-bound writer) -> GB/s, roofline
  decode : W warm-up + K decode steps dkv_classify -> dkv_compact_alloc -> dkv_quant_write; between timed
           steps (untimed) the significance drift (attention stand-in), next-step inputs and a 256 MiB L2
           flush; every 10th step frees one request first (its compact_alloc recycles ~37k pages) and
           re-admits it after.  value = mean µs of dkv_compact_alloc per decode step (max over ranks).
  e2e    : K decode steps, each ONE C-ABI call with pinned HOST buffers (dkv_decode_step_host: cand_sig and new K/V copied in,
           the decisions copied out, all inside the timed region).
At N > 1 each step also all-reduces the pool's int64[4] admission counters (MIN) over NCCL on a side
stream (one-step lag), the only collective of the path.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

CONFIGS = {
    "llama3_8b": dict(R=64, Ly=32, H=8, d=128, prompt=4096, M=8192, W=64, Ch=16, Cl=32, P=1 << 22,
                      alpha_h=1.0, alpha_l=0.02, mix=(0.35, 0.45, 0.20), seed=2, G=4),
    "tiny": dict(R=4, Ly=2, H=4, d=64, prompt=64, M=128, W=16, Ch=16, Cl=32, P=1024,
                 alpha_h=1.0, alpha_l=0.02, mix=(0.35, 0.45, 0.20), seed=1, G=4),
}
METRIC = "µs per decode-step compact+alloc (64 req×32L×8H); quant-write GB/s vs HBM peak, 1/2/4/8 GPU"
# the e2e key of both arms: one whole decode step (classify + compact_alloc + quant_write) through the public API
E2E_UNIT = "us per decode step (classify + compact_alloc + quant_write through the public API)"


# ----------------------------------------------------------------------------------------- distributed
DIST = {"backend": None, "red_device": "cuda"}


def dist_init(shared_device=False):
    """One rank per GPU from the torchrun environment (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*).  NCCL carries
    the per-step count all-reduce (NCCL_DEBUG=INFO, subsystem INIT, prints each communicator's nranks to
    stderr); with --shared-device (more ranks than GPUs) the ranks share GPUs and reduce over gloo."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    dev = local % max(ndev, 1) if shared_device else local
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        if shared_device and ndev < world:
            dist.init_process_group("gloo")
            DIST.update(backend="gloo", red_device="cpu")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
            DIST.update(backend="nccl", red_device="cuda")
    return rank, world, dev


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _reduce(x: float, world: int, op) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=DIST["red_device"])
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x: float, world: int) -> float:
    import torch.distributed as dist
    return _reduce(x, world, dist.ReduceOp.MAX if world > 1 else None)


def sum_over_ranks(x: float, world: int) -> float:
    import torch.distributed as dist
    return _reduce(x, world, dist.ReduceOp.SUM if world > 1 else None)


# ----------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/dkv_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------------------- workload
class Workload:
    """Synthetic inputs of one GPU's shard, generated on the device from counters (synth/)."""

    def __init__(self, c, rank, world, device, strong=False):
        self.c = c
        self.world = world
        assert c["H"] % world == 0
        self.Hl = c["H"] // world
        # weak scaling (default): the global batch grows with N, per-GPU units fixed; strong: the global batch is
        # fixed and each GPU's pool holds H/N of its heads
        self.R = c["R"] if strong else c["R"] * world
        self.shape = synth.Shape(self.R, c["Ly"], self.Hl, H_total=c["H"], h0=rank * self.Hl)
        self.LyH = c["Ly"] * self.Hl
        self.U = self.R * self.LyH
        self.device = device
        ug = self.shape.global_units(list(range(self.R)), device="cpu")
        mh, ml = synth.unit_mix(c["seed"], ug, c["mix"], Ly=c["Ly"], Ht=c["H"])
        self.ug = ug.to(device)
        self.mix_h, self.mix_l = mh.to(device), ml.to(device)

    def prefill_inputs(self, T):
        c, dev = self.c, self.device
        sig = torch.empty((self.R, self.LyH, T), dtype=torch.float32, device=dev)
        k = torch.empty((self.R, self.LyH, T, c["d"]), dtype=torch.float16, device=dev)
        v = torch.empty_like(k)
        step = max(1, (64 if dev.type == "cuda" else 4) // max(1, T // 512))
        for r in range(self.R):
            sig[r] = synth.prefill_sig(c["seed"], self.ug[r], T, c["alpha_h"], c["alpha_l"], self.mix_h[r],
                                       self.mix_l[r])
            for j0 in range(0, self.LyH, step):
                g = self.ug[r, j0:j0 + step]
                k[r, j0:j0 + step] = synth.kv_values(c["seed"], synth.S_KEY, g, 0, T, c["d"])
                v[r, j0:j0 + step] = synth.kv_values(c["seed"], synth.S_VAL, g, 0, T, c["d"])
        return sig, k, v

    def decode_inputs(self, seq_len_host, active_host):
        c = self.c
        N = torch.as_tensor(np.where(active_host, seq_len_host + 1, 0), dtype=torch.int64, device=self.device)
        N = N.view(-1, 1).expand(-1, self.LyH).reshape(-1)
        ug = self.ug.reshape(-1)
        cand = synth.decode_sig(c["seed"], ug, N, c["W"], c["alpha_h"], c["alpha_l"], self.mix_h.reshape(-1),
                                self.mix_l.reshape(-1))
        k, v = synth.new_token_kv(c["seed"], ug, (N - 1).clamp(min=0), c["d"])
        return cand.contiguous(), k.contiguous(), v.contiguous()


def bulk_bytes_counts(nh, nl, kept, nw, geom, d):
    """Algorithmic bytes of one dkv_quant_write(PREFILL), SURVEY §8(d) accounting: a kept token reads its K and
    V (2·d fp16 = 512 B at d = 128) and writes its codes + {s, z} K/V metadata + score + position (High K8V4:
    128 + 64 + 4 + 4 + 4 + 4 = 208 B -> 720 B; Low K4V2: 112 B -> 624 B); a pruned token moves nothing; a
    window token reads 2·d fp16 and writes them to the window (1024 B at d = 128)."""
    hb = 4 * d + geom[1]["k_row"] + geom[1]["v_row"] + 16
    lb = 4 * d + geom[2]["k_row"] + geom[2]["v_row"] + 16
    return nh * hb + nl * lb + nw * 8 * d, dict(high=nh, low=nl, pruned=kept - nh - nl, window=nw)


def bulk_bytes(pool, geom, W, d, T, units):
    """bulk_bytes_counts for the pool's current contents after an admission of `units` prompts of T tokens"""
    v = pool.views()
    nh = int(v["n_h"].sum().item())
    nl = int(v["n_l"].sum().item())
    return bulk_bytes_counts(nh, nl, units * max(T - W, 0), units * min(W, T), geom, d)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_fp32_peak():
    """FP32 FFMA peak for the attention kernel's ALU roofline: measured by tools/fmabench.cu on a B200
    (profiles/fp32_peak.json), else the nominal 148 SMs x 128 FMA/clk x 2 x 1.965 GHz."""
    p = os.path.join(ROOT, "profiles", "fp32_peak.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["fp32_tflops"]), "measured (profiles/fp32_peak.json, tools/fmabench.cu)"
    return 148 * 128 * 2 * 1.965e9 / 1e12, "nominal (148 SMs x 128 FP32 lanes x 2 x 1965 MHz)"


def load_traffic():
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of each kernel, from the committed
    `ncu --set full` summaries (profiles/traffic.json, written by tools/make_profiles.py)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return lambda k: None
    with open(p) as f:
        j = json.load(f)

    def get(kernel):
        for name, rec in j.items():
            if name.split("<")[0] == kernel:
                return int(rec["bytes_per_launch"])
        return None
    return get


def scatter_note(achieved):
    """The scan reads one 64-B (high page) or 128-B (low page) score segment per page, scattered over the pool: its
    ceiling is the measured random-segment gather rate (profiles/scatter_peaks.json, tools/scatter_bench.cu), not the
    streaming HBM peak."""
    p = os.path.join(ROOT, "profiles", "scatter_peaks.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    return {"random_64B_gbs": j["random_64B_gbs"], "random_128B_gbs": j["random_128B_gbs"],
            "frac_of_64B": round(achieved / j["random_64B_gbs"], 3), "frac_of_128B": round(achieved / j["random_128B_gbs"], 3),
            "source": j["source"]}


def stream_mix_note(achieved):
    """The bulk writer's DRAM mix is ~3.2 bytes read per byte written (ncu): context for its roofline fraction is
    the measured rate of contiguous read:write streams at 3:1 and 4:1 on the same kind of box
    (profiles/scatter_peaks.json); the reported `frac` stays against MEASURED_PEAKS.json."""
    p = os.path.join(ROOT, "profiles", "scatter_peaks.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    if "rw_stream_3to1_gbs" not in j:
        return None
    return {"rw_stream_3to1_gbs": j["rw_stream_3to1_gbs"], "rw_stream_4to1_gbs": j["rw_stream_4to1_gbs"],
            "frac_of_3to1": round(achieved / j["rw_stream_3to1_gbs"], 3), "source": j["source"]}


# ----------------------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    from paper_2412_03131_b200 import Pool
    from paper_2412_03131_b200 import dkv as D

    c = CONFIGS[args.config]
    dev = torch.device("cuda", local)
    wl = Workload(c, rank, world, dev, strong=args.strong)
    cfg = D.make_config(wl.R, c["Ly"], wl.Hl, c["d"], c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"],
                        alpha_h=c["alpha_h"], alpha_l=c["alpha_l"], tile_units=args.tile_units,
                        q_per_kv=c.get("G", 0))
    pool = Pool(cfg, device=dev)
    geom = pool.geom()
    T = c["prompt"]
    sig, kk, vv = wl.prefill_inputs(T)
    k16, v16 = kk.view(torch.int16), vv.view(torch.int16)
    reqs = list(range(wl.R))
    lens = [T] * wl.R
    dec = pool.new_decisions()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    launches = 0

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def empty_step():
        """decode step used only to recycle PENDING_FREE requests (no ACTIVE request, untimed)"""
        z = torch.zeros(wl.U, dtype=torch.float32, device=dev)
        zk = torch.zeros((wl.U, c["d"]), dtype=torch.int16, device=dev)
        pool.classify_decode(z, dec)
        pool.compact_alloc(dec)
        pool.quant_write_decode(dec, zk, zk, z)

    # ---------------- bulk phase: K rounds of prefill quant-write of the whole batch
    sampler = ClockSampler(local)
    bulk_ms = []
    nrounds = args.warmup + args.steps
    sampler.start()
    t_wall0 = time.time()
    for i in range(nrounds):
        if i > 0:
            pool.free(reqs)
            empty_step()
        pool.classify_prefill(reqs, lens, sig)
        pool.compact_alloc(None)
        flush.zero_()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = ev(), ev()
        torch.cuda._sleep(200_000)                         # see the decode phase: time device execution
        e0.record()
        pool.quant_write_prefill(k16, v16, sig)
        e1.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            bulk_ms.append(e0.elapsed_time(e1))
            launches += 2                                  # quant_prefill_kernel + finish_prefill_kernel
    st, stats = pool.query()
    assert st == 0, f"device status {st} after prefill"
    bbytes, bmix = bulk_bytes(pool, geom, c["W"], c["d"], T, wl.U)
    bulk_mean = statistics.mean(bulk_ms)
    bulk_max = max_over_ranks(bulk_mean, world)

    # ---------------- decode phase
    from paper_2412_03131_b200.admission import Admission, prefill_page_bound
    seq = np.full(wl.R, T, np.int64)
    active = np.ones(wl.R, bool)
    nccl = DIST["backend"] == "nccl"
    side = torch.cuda.Stream(device=dev) if world > 1 and nccl else None
    v0 = pool.views()
    stats_view = v0["stats"]
    red = torch.empty(4, dtype=torch.int64, device=dev if nccl else "cpu")
    comp_us, cls_us, qw_us, step_us, cls_bytes = [], [], [], [], []
    ar_us, ar_hidden = [], []
    realized = {"demand": [], "freed": [], "downgrades": [], "pruned_victims": [], "oom": 0}
    # SURVEY §8e admission: a freed request's slot is re-admitted only when EVERY GPU has room for its shard's
    # prefill bound plus the decode reserve (one page per unit), judged on the MIN-reduced counters
    adm = Admission(decode_reserve=wl.U)
    bound = prefill_page_bound(T, c["W"], c["Ch"], wl.LyH)
    waiting, admitted_n, deferred_n = [], 0, 0
    # launch floor: event -> trivial kernel -> event, measured the same way as the step kernels
    floor_us = []
    for _ in range(20):
        torch.cuda.synchronize()
        f0, f1 = ev(), ev()
        torch.cuda._sleep(200_000)
        f0.record()
        torch.cuda._sleep(0)
        f1.record()
        torch.cuda.synchronize()
        floor_us.append(f0.elapsed_time(f1) * 1e3)
    floor = float(np.median(floor_us))
    freed_steps = 0
    total_steps = args.warmup + args.steps
    for s in range(total_steps):
        timed = s >= args.warmup
        # untimed: attention stand-in (significance drift), inputs, churn, L2 flush
        v = pool.views()
        synth.apply_drift(c["seed"], s, wl.shape, v["pages"], v["table"], v["n_h"], v["n_l"],
                          {k_: (geom[k_]["C"], geom[k_]["off_score"], geom[k_]["off_pos"]) for k_ in (1, 2)}, pool.L)
        churn = timed and (s - args.warmup) % 10 == 5
        if churn:
            r = (s * 7) % wl.R
            pool.free([r])
            active[r] = False
            waiting.append(r)
            freed_steps += 1
        cand, nk, nv = wl.decode_inputs(seq, active)
        nh0, nl0 = v["n_h"].clone(), v["n_l"].clone()
        flush.zero_()
        torch.cuda.synchronize()
        barrier(world)
        e = [ev() for _ in range(4)]
        ar = [ev(), ev()]
        # a ~100 µs device-side spin ahead of the step lets the host enqueue all three ABI calls before the
        # GPU reaches e[0], so the events time device execution, not Python/ctypes submission latency
        # (e2e below keeps the host path in its timed region)
        torch.cuda._sleep(200_000)
        e[0].record()
        pool.classify_decode(cand, dec)
        e[1].record()
        pool.compact_alloc(dec)
        e[2].record()
        if side is not None:                                # count all-reduce over NCCL, overlapped with quant_write
            import torch.distributed as dist
            side.wait_event(e[2])
            with torch.cuda.stream(side):
                ar[0].record(side)
                red.copy_(stats_view)
                dist.all_reduce(red, op=dist.ReduceOp.MIN)
                ar[1].record(side)
        pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), cand)
        e[3].record()
        torch.cuda.synchronize()
        if side is None:                                    # one rank, or gloo (--shared-device): after the step
            red.copy_(stats_view)
            if world > 1:
                import torch.distributed as dist
                dist.all_reduce(red, op=dist.ReduceOp.MIN)
        seq[active] += 1
        # Ctrl as int64: start, free, {status, oom_count}, ticket, arrive, last_demand, last_freed
        ct = pool.arena[int(pool.layout.off_ctrl):int(pool.layout.off_ctrl) + 56].view(torch.int64).cpu().numpy()
        # admission on the reduced counters (identical on every rank, so every rank decides the same)
        for r in list(waiting):
            if adm.admit(red.cpu(), bound):
                pool.classify_prefill([r], [T], sig[r:r + 1])   # re-admit (untimed prefill of a 4096-token prompt)
                pool.compact_alloc(None)
                pool.quant_write_prefill(k16[r:r + 1], v16[r:r + 1], sig[r:r + 1])
                seq[r] = T
                active[r] = True
                waiting.remove(r)
                admitted_n += 1
            else:
                deferred_n += 1
        if timed:
            cls_us.append(e[0].elapsed_time(e[1]) * 1e3)
            comp_us.append(e[1].elapsed_time(e[2]) * 1e3)
            qw_us.append(e[2].elapsed_time(e[3]) * 1e3)
            step_us.append(e[0].elapsed_time(e[3]) * 1e3)
            launches += 3 + (1 if churn else 0)             # classify, compact_alloc, quant_decode (+ recycle)
            if side is not None:                            # count all-reduce latency; hidden if it ended in the step
                ar_us.append(ar[0].elapsed_time(ar[1]) * 1e3)
                ar_hidden.append(e[0].elapsed_time(ar[1]) <= e[0].elapsed_time(e[3]))
            d16 = dec.view(torch.uint8).view(-1, 16).cpu().numpy()
            tc = d16[:, 0]
            sec = np.where(tc == 1, nh0.cpu().numpy(), np.where(tc == 2, nl0.cpu().numpy(), 0)).astype(np.int64)
            C = np.where(tc == 1, geom[1]["C"], geom[2]["C"])
            cls_bytes.append(int((4 * sec + 4 * ((sec + C - 1) // C)).sum() + 28 * wl.U))
            realized["demand"].append(int(ct[5]))
            realized["freed"].append(int(ct[6]))
            realized["downgrades"].append(int((d16[:, 1] == 2).sum()))
            realized["pruned_victims"].append(int((d16[:, 1] == 3).sum()))
            realized["oom"] += int(int(ct[2]) & 0xFFFFFFFF == (-3 & 0xFFFFFFFF))
    st, stats = pool.query()
    assert st == 0, f"device status {st} after decode"
    wall = time.time() - t_wall0
    clocks = sampler.stop()
    # validation, outside every timed region: the device audit of the pool's invariants after the decode phase
    audit = pool.audit()
    audit["sound"] = bool(audit["used_pages"] + audit["free_pages"] == c["P"] and
                          all(v == 0 for k, v in audit.items() if k not in ("used_pages", "free_pages")))

    # ---------------- e2e: same decode step through the C ABI with host buffers
    e2e_us = []
    pin_c = torch.empty((args.steps, wl.U), dtype=torch.float32).pin_memory()
    # K and V of a step side by side in one pinned buffer: one 8.4 MB H2D copy per step instead of two
    pin_kv = torch.empty((args.steps, 2, wl.U, c["d"]), dtype=torch.int16).pin_memory()
    pin_k, pin_v = pin_kv[:, 0], pin_kv[:, 1]
    pin_dec = torch.empty((wl.U, 4), dtype=torch.int32).pin_memory()
    for i in range(args.steps):
        cand, nk, nv = wl.decode_inputs(seq + i, active)
        pin_c[i].copy_(cand)
        pin_k[i].copy_(nk.view(torch.int16))
        pin_v[i].copy_(nv.view(torch.int16))
    # one C-ABI call per step with HOST buffers (dkv_decode_step_host): the library copies the significance
    # and the new tokens' K/V (8.4 MB at this config; on its own copy stream, overlapping classify +
    # compact_alloc; quant_write waits for it), runs the three kernels' calls and copies the decisions back
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = ev(), ev()
        e0.record()
        pool.decode_step_host(pin_c[i], pin_kv[i], pin_dec)
        e1.record()
        torch.cuda.synchronize()
        e2e_us.append(e0.elapsed_time(e1) * 1e3)
    st, stats = pool.query()
    assert st == 0, f"device status {st} after e2e"
    seq[active] += args.steps
    # the host link in the same run: the step's K/V bytes alone (one pinned H2D copy), and a 256 MiB copy
    link = {}
    kv_dev = torch.empty_like(pin_kv[0], device=dev)
    big_h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    big_d = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for name, (src, dst) in (("kv", (pin_kv[0], kv_dev)), ("big", (big_h, big_d))):
        ts = []
        for i in range(4):
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            if i:
                ts.append(e0.elapsed_time(e1) * 1e3)
        link[name] = statistics.mean(ts)
    h2d_link = {"step_kv_copy_us": round(link["kv"], 1), "step_kv_bytes": int(pin_kv[0].numel() * 2),
                "link_gbs_256mib": round((256 << 20) / (link["big"] * 1e-6) / 1e9, 1)}
    del big_h, big_d, kv_dev

    # ---------------- NEXT-2: decode steps driven by the attention kernel's significance
    next2 = None
    if args.next2 and c.get("G", 0) > 0:
        G, d = c["G"], c["d"]
        gen = torch.Generator(device=dev)
        gen.manual_seed(c["seed"] + rank)
        qbuf = torch.empty((wl.U, G, d), dtype=torch.float16, device=dev)
        obuf = torch.empty((wl.U, G, d), dtype=torch.float32, device=dev)
        v = pool.views()
        qbuf.normal_(generator=gen)
        pool.attend(qbuf.view(torch.int16), obuf)                 # primes the window significance + minima

        def run_next2(attend_fn):
            nonlocal launches
            att_us, cls2_us, step2_us, att_bytes, att_flops = [], [], [], [], []
            for s in range(args.warmup + args.steps):
                timed = s >= args.warmup
                cand, nk, nv = wl.decode_inputs(seq, active)
                qbuf.normal_(generator=gen)
                flush.zero_()
                torch.cuda.synchronize()
                barrier(world)
                e = [ev() for _ in range(5)]
                torch.cuda._sleep(200_000)
                e[0].record()
                pool.classify_decode(None, dec)
                e[1].record()
                pool.compact_alloc(dec)
                e[2].record()
                pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), None)
                e[3].record()
                attend_fn(qbuf.view(torch.int16), obuf)
                e[4].record()
                torch.cuda.synchronize()
                seq[active] += 1
                if timed:
                    cls2_us.append(e[0].elapsed_time(e[1]) * 1e3)
                    att_us.append(e[3].elapsed_time(e[4]) * 1e3)
                    step2_us.append(e[0].elapsed_time(e[4]) * 1e3)
                    launches += 4
                    # algorithmic bytes of one attention pass: every stored token's K/V codes, metadata, position and
                    # score (read + write back), every window token's fp16 K/V and significance (read + write),
                    # the queries and the output
                    nh1, nl1 = v["n_h"].long(), v["n_l"].long()
                    gh_, gl_ = geom[1], geom[2]
                    per_h = gh_["k_row"] + gh_["v_row"] + 8 + 4 + 4 + 4
                    per_l = gl_["k_row"] + gl_["v_row"] + 8 + 4 + 4 + 4
                    nwin = min(c["W"], int(seq.max()))
                    att_bytes.append(int((nh1.sum() * per_h + nl1.sum() * per_l).item())
                                     + wl.U * (nwin * (4 * d + 8) + G * d * 2 + G * d * 4))
                    # algorithmic flops: per token the G logit and G output dot products over d elements (2 G d
                    # fma); a stored token's key and value dequantization adds 2 d fma
                    n_stored = int((nh1.sum() + nl1.sum()).item())
                    n_win = wl.U * nwin
                    att_flops.append(2 * ((n_stored + n_win) * 2 * G * d + n_stored * 2 * d))
            st, _ = pool.query()
            assert st == 0, f"device status {st} after the NEXT-2 steps"
            return att_us, cls2_us, step2_us, att_bytes, att_flops

        att_us, cls2_us, step2_us, att_bytes, att_flops = run_next2(lambda q_, o_: pool.attend(q_, o_))
        tc_us, tc_cls_us, tc_step_us, tc_bytes, _ = run_next2(lambda q_, o_: pool.attend_tc(q_, o_))
        tc_mean = max_over_ranks(statistics.mean(tc_us), world)
        tc_gbs = statistics.mean(tc_bytes) / (statistics.mean(tc_us) * 1e-6) / 1e9
        # the same batch's KV as FP16 (2 x d x 2 bytes per stored or window token) read at the measured HBM peak: the
        # time an FP16 attention needs at roofline (the paper's comparison)
        fp16_bytes = (int((v["n_h"].long().sum() + v["n_l"].long().sum()).item())
                      + wl.U * min(c["W"], int(seq.max()))) * 4 * d
        fp16_us = fp16_bytes / (load_peaks()[0] * 1e9) * 1e6
        att_mean = max_over_ranks(statistics.mean(att_us), world)
        att_gbs = statistics.mean(att_bytes) / (statistics.mean(att_us) * 1e-6) / 1e9
        next2 = {"attend_us": round(att_mean, 1), "attend_gbs": round(att_gbs, 1),
                 "attend_frac_of_hbm_peak": round(att_gbs / load_peaks()[0], 4),
                 "attend_algorithmic_bytes": int(statistics.mean(att_bytes)),
                 "classify_fused_us": round(max_over_ranks(statistics.mean(cls2_us), world), 3),
                 "step_us": round(max_over_ranks(statistics.mean(step2_us), world), 1),
                 "q_per_kv": G,
                 # the paper's only figure for this path: memory management < 0.9 % of a generation step (L40,
                 # P:859); here the step is the manager's three calls + the compressed-cache attention
                 "manager_share_of_step": round(1.0 - statistics.mean(att_us) / statistics.mean(step2_us), 4),
                 "roofline": {"kernel": "attend_kernel", "bound": "alu",
                              "achieved": round(statistics.mean(att_flops) / (statistics.mean(att_us) * 1e-6) / 1e12, 2),
                              "peak": round(load_fp32_peak()[0], 2), "peak_source": load_fp32_peak()[1],
                              "unit": "TFLOP/s",
                              "frac": round(statistics.mean(att_flops) / (statistics.mean(att_us) * 1e-6) / 1e12
                                            / load_fp32_peak()[0], 4),
                              "algorithmic_flops": int(statistics.mean(att_flops)),
                              "note": "exact fp32 fma chains (Q31/Q32) on CUDA cores; the kernel also issues the "
                                      "code->float conversions, softmax and significance work, so it is bound by "
                                      "instruction issue (ncu: profiles/*prof_attend*)"},
                 "note": "dkv_attend (NEXT-2) supplies significance; classify takes its victims from the "
                         "attention kernel's section minima (no scan)"}
        next2["tc"] = {"kernel": "attend_tc_kernel (dkv_attend_tc: mma.sync on the integer codes, fp32 accumulation)",
                       "attend_us": round(tc_mean, 1),
                       "classify_fused_us": round(max_over_ranks(statistics.mean(tc_cls_us), world), 3),
                       "step_us": round(max_over_ranks(statistics.mean(tc_step_us), world), 1),
                       "manager_share_of_step": round(1.0 - statistics.mean(tc_us) / statistics.mean(tc_step_us), 4),
                       "roofline": {"bound": "hbm", "achieved": round(tc_gbs, 1), "peak": load_peaks()[0],
                                    "unit": "GB/s", "frac": round(tc_gbs / load_peaks()[0], 4),
                                    "algorithmic_bytes": int(statistics.mean(tc_bytes)),
                                    "traffic": load_traffic()("attend_tc_kernel"), "traffic_unit": "bytes per launch"},
                       "fp16_attention_at_roofline_us": round(fp16_us, 1),
                       "speedup_vs_fp16_roofline": round(fp16_us / statistics.mean(tc_us), 3),
                       "note": "FP16 reference: the same tokens' K and V as fp16 (4 d bytes each) read at the measured "
                               "HBM peak; the paper reports 1.7x for K8V8 over FP16 (P:896-900)"}

    # ---------------- CUDA graph: GRAPH_STEPS decode steps captured once (dkv_decode_graph_create) and replayed;
    # per-step inputs [GRAPH_STEPS][U][d] (840 MB at this config, >> L2) already in HBM.  No L2 flush between the
    # steps of a replay: it is the steady state of back-to-back decode steps.
    from paper_2412_03131_b200 import dkv as D
    # the replays (two per PDL / plain graph, one event graph) must stay within max_seq_len
    GS = max(1, min(100, (c["M"] - int(seq.max()) - 4 * (args.warmup + args.steps) - 8) // 6))
    gsig = torch.empty((GS, wl.U), dtype=torch.float32, device=dev)
    gk = torch.empty((GS, wl.U, c["d"]), dtype=torch.int16, device=dev)
    gv = torch.empty_like(gk)
    for t in range(GS):
        cand, nk, nv = wl.decode_inputs(seq + t, active)
        gsig[t].copy_(cand)
        gk[t].copy_(nk.view(torch.int16))
        gv[t].copy_(nv.view(torch.int16))
    gdec = pool.new_decisions()
    graph_pdl = pool.decode_graph(GS, gsig, gk, gv, gdec, D.DKV_GRAPH_PDL)
    graph_ev = pool.decode_graph(GS, gsig, gk, gv, gdec, D.DKV_GRAPH_EVENTS)
    graph_plain = pool.decode_graph(GS, gsig, gk, gv, gdec, 0)
    graph_us = {}
    for name, gr in (("pdl", graph_pdl), ("plain", graph_plain)):
        for rep in range(2):                                 # one untimed replay, one timed
            flush.zero_()
            torch.cuda.synchronize()
            barrier(world)
            g0, g1 = ev(), ev()
            torch.cuda._sleep(200_000)
            g0.record()
            gr.launch()
            g1.record()
            torch.cuda.synchronize()
            seq[active] += GS
            launches += 3 * GS if rep else 0
        graph_us[name] = g0.elapsed_time(g1) * 1e3 / GS
    flush.zero_()
    graph_ev.launch()
    torch.cuda.synchronize()
    seq[active] += GS
    kms = graph_ev.kernel_ms() * 1e3                         # [GS][3] us: classify, compact_alloc, quant_write
    st, _ = pool.query()
    assert st == 0, f"device status {st} after the graph replays"
    for gr in (graph_pdl, graph_ev, graph_plain):
        gr.close()
    del gsig, gk, gv
    # a ONE-step graph replayed per step, with the same untimed drift + L2 flush between steps as the eager decode
    # phase: its device time is directly comparable to decode_step_us.step
    s_sig = torch.empty(wl.U, dtype=torch.float32, device=dev)
    s_k = torch.empty((wl.U, c["d"]), dtype=torch.int16, device=dev)
    s_v = torch.empty_like(s_k)
    graph1 = pool.decode_graph(1, s_sig, s_k, s_v, gdec, D.DKV_GRAPH_PDL)
    g1_us = []
    for s_ in range(args.warmup + args.steps):
        v = pool.views()
        synth.apply_drift(c["seed"], 1000 + s_, wl.shape, v["pages"], v["table"], v["n_h"], v["n_l"],
                          {k_: (geom[k_]["C"], geom[k_]["off_score"], geom[k_]["off_pos"]) for k_ in (1, 2)}, pool.L)
        cand, nk, nv = wl.decode_inputs(seq, active)
        s_sig.copy_(cand)
        s_k.copy_(nk.view(torch.int16))
        s_v.copy_(nv.view(torch.int16))
        flush.zero_()
        torch.cuda.synchronize()
        barrier(world)
        g0, g1 = ev(), ev()
        torch.cuda._sleep(200_000)
        g0.record()
        graph1.launch()
        g1.record()
        torch.cuda.synchronize()
        seq[active] += 1
        if s_ >= args.warmup:
            g1_us.append(g0.elapsed_time(g1) * 1e3)
            launches += 3
    graph1.close()
    st, _ = pool.query()
    assert st == 0, f"device status {st} after the one-step graph replays"
    graph = {"one_step_graph_us": round(max_over_ranks(statistics.mean(g1_us), world), 3),
             "one_step_graph_us_p50": round(float(np.percentile(g1_us, 50)), 3),
             "steps_per_graph": GS, "graph_step_us": round(max_over_ranks(graph_us["pdl"], world), 3),
             "graph_step_us_no_pdl": round(max_over_ranks(graph_us["plain"], world), 3),
             "in_graph_kernel_us": {nm: {"mean": round(float(kms[:, j].mean()), 3),
                                         "p50": round(float(np.percentile(kms[:, j], 50)), 3),
                                         "p99": round(float(np.percentile(kms[:, j], 99)), 3)}
                                    for j, nm in enumerate(("classify", "compact_alloc", "quant_write"))},
             "note": "one_step_graph_us: a 1-step graph (PDL) replayed per step with the eager phase's drift and L2 "
                     "flush in between (compare decode_step_us.step); graph_step_us = device time of one replay of a "
                     "100-step graph (PDL between kernels) / 100, steady state (no drift, no L2 flush inside a "
                     "replay: more ties in the scan), inputs 840 MB per replay; in_graph_kernel_us from the same "
                     "100-step graph with an event node around every kernel (no PDL)"}

    # ---------------- recycle micro-benchmark: free 1 / 8 / 32 requests, then one decode step whose
    # dkv_compact_alloc recycles all their pages (~37k / 300k / 1.2M page IDs at this config)
    recycle = {}
    if wl.R >= 32:
        for kq in (1, 8, 32):
            reqs_k = [r for r in range(wl.R) if active[r]][:kq]
            r0 = reqs_k[0]
            if reqs_k != list(range(r0, r0 + kq)):
                continue
            pool.free(reqs_k)
            active[reqs_k] = False
            cand, nk, nv = wl.decode_inputs(seq, active)
            flush.zero_()
            torch.cuda.synchronize()
            e = [ev() for _ in range(3)]
            torch.cuda._sleep(200_000)
            e[0].record()
            pool.classify_decode(cand, dec)
            e[1].record()
            pool.compact_alloc(dec)
            e[2].record()
            pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), cand)
            torch.cuda.synchronize()
            launches += 4
            seq[active] += 1
            ct = pool.arena[int(pool.layout.off_ctrl):int(pool.layout.off_ctrl) + 56].view(torch.int64).cpu().numpy()
            recycle[str(kq)] = {"compact_alloc_us": round(e[1].elapsed_time(e[2]) * 1e3, 2),
                                "recycled_pages": int(ct[6])}
            pool.classify_prefill(reqs_k, [T] * kq, sig[r0:r0 + kq])
            pool.compact_alloc(None)
            pool.quant_write_prefill(k16[r0:r0 + kq], v16[r0:r0 + kq], sig[r0:r0 + kq])
            seq[reqs_k] = T
            active[reqs_k] = True
        st, _ = pool.query()
        assert st == 0, f"device status {st} after the recycle micro-benchmark"

    # ---------------- aggregate (max over ranks)
    comp_mean = max_over_ranks(statistics.mean(comp_us), world)
    step_mean = max_over_ranks(statistics.mean(step_us), world)
    cls_mean = max_over_ranks(statistics.mean(cls_us), world)
    qw_mean = max_over_ranks(statistics.mean(qw_us), world)
    e2e_mean = max_over_ranks(statistics.mean(e2e_us), world)
    bulk_gbs_rank = bbytes / (bulk_mean * 1e-3) / 1e9
    agg_bulk_gbs = sum_over_ranks(bbytes, world) / (bulk_max * 1e-3) / 1e9
    peak, peak_src = load_peaks()
    traffic = load_traffic()
    cls_gbs = statistics.mean(cls_bytes) / (statistics.mean(cls_us) * 1e-6) / 1e9
    out = {
        "metric": METRIC,
        "value": round(comp_mean, 3),
        "unit": "us",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_mean / 1e3, 6),
        "higher_is_better": False,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None,
        "dtype": "fp16 in / u8 codes (fp32 quantizer arithmetic, int32 scans)",
        "data": "synthetic (seeded counter-based significance / K / V, synth/)",
        "config": {
            "workload": f"{args.config}: Llama-3-8B KV shape, {c['R']}x{world} req x {c['Ly']} layers x {c['H']} KV heads "
                        f"(sharded {world}-way), d {c['d']}, prompt {T}, M {c['M']}, W {c['W']}, K8V4/16-token + "
                        f"K4V2/32-token pages, {c['P']} pages per GPU, alpha {c['alpha_h']}/{c['alpha_l']}",
            "units_per_gpu": wl.U,
            "global_batch": wl.R,
            "parallelism": f"kv-head shard x{world} (independent pools)",
            "l2": "flushed between timed steps (256 MiB write); bulk inputs 32 GiB >> L2",
        },
        "decode_step_us": {"classify": round(cls_mean, 3), "compact_alloc": round(comp_mean, 3),
                           "quant_write": round(qw_mean, 3), "step": round(step_mean, 3),
                           **{f"{name}_p{q}": round(float(np.percentile(xs, q)), 3)
                              for name, xs in (("classify", cls_us), ("compact_alloc", comp_us), ("quant_write", qw_us))
                              for q in (50, 99)},
                           "percentile_note": f"over {len(comp_us)} timed steps (p99 of so few samples is near the max)",
                           "launch_floor": round(floor, 3),
                           "recycle_steps": freed_steps},
        # what each step actually did (means over the timed steps)
        "realized_per_step": {"demand_pages": round(statistics.mean(realized["demand"]), 1),
                              "freed_pages": round(statistics.mean(realized["freed"]), 1),
                              "downgrades": round(statistics.mean(realized["downgrades"]), 1),
                              "pruned_victims": round(statistics.mean(realized["pruned_victims"]), 1),
                              "oom_steps": realized["oom"]},
        "admission": {"rule": "admit iff MIN over GPUs of free pages >= prefill bound + one page per unit "
                              "(paper_2412_03131_b200/admission.py, on the all-reduced counters)",
                      "admitted": admitted_n, "deferred_checks": deferred_n, "prefill_bound_pages": bound},
        "dist": {"backend": DIST["backend"], "world": world,
                 "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if DIST["backend"] == "nccl" else None},
        "quant_write": {"gbs": round(agg_bulk_gbs, 1), "gbs_per_gpu": round(bulk_gbs_rank, 1),
                        "ms": round(bulk_max, 3), "ms_rounds": [round(x, 3) for x in bulk_ms], "algorithmic_bytes_per_gpu": bbytes, "token_mix": bmix,
                        "frac_of_hbm_peak": round(bulk_gbs_rank / peak, 4)},
        "roofline": {"kernel": "quant_prefill_kernel (dkv_quant_write PREFILL, bulk writer)", "bound": "hbm",
                     "achieved": round(bulk_gbs_rank, 1), "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(bulk_gbs_rank / peak, 4),
                     "traffic": traffic("quant_prefill_kernel"), "traffic_unit": "bytes per launch",
                     "access_pattern": stream_mix_note(bulk_gbs_rank)},
        "roofline_decode": {"kernel": "classify_decode_kernel", "bound": "hbm", "achieved": round(cls_gbs, 1),
                            "peak": peak, "unit": "GB/s", "frac": round(cls_gbs / peak, 4),
                            "algorithmic_bytes": int(statistics.mean(cls_bytes)),
                            "traffic": traffic("classify_decode_kernel"), "traffic_unit": "bytes per launch",
                            "access_pattern": scatter_note(cls_gbs)},
        "e2e": {"value": round(e2e_mean, 3), "unit": E2E_UNIT,
                "h2d_bytes_per_step": wl.U * (4 + 2 * 2 * c["d"]), "d2h_bytes_per_step": wl.U * 16,
                "h2d_link": h2d_link},
        "audit": audit,
        "graph": graph if GS >= 10 else None,
        "next2": next2,
        # §8e: the per-step MIN all-reduce of the admission counters (N > 1): its latency on the side stream and
        # the fraction of steps in which it finished inside the step (hidden behind quant_write)
        "allreduce": ({"us": round(max_over_ranks(statistics.mean(ar_us), world), 2),
                       "hidden_frac": round(sum(ar_hidden) / len(ar_hidden), 3), "bytes": 32}
                      if ar_us else None),
        "recycle_microbench": recycle,
        # the paper's own figure for this path (other hardware: context, not a target): the whole memory manager
        # is < 0.2 % (prompt) / < 0.9 % (generation) of step latency on L40 inside vLLM
        "paper_context": {"manager_share_of_step_L40": {"prompt": "< 0.2 %", "generation": "< 0.9 %"},
                          "cite": "PAPER.md:853-859 (§7.2 Memory Management Overhead)"},
        "gpu_launches": launches,
        "clocks": clocks,
        "wall_s": round(wall, 1),
    }
    return out


# ----------------------------------------------------------------------------------------- oracle arm
def run_oracle_sample(args, sample_requests=1, steps=None):
    """The serial C oracle (oracle/, as it stands) on a bounded sample of the same workload: the first
    `sample_requests` requests (all their layers and heads), prefill + decode steps; times scaled to the
    full per-GPU batch by the unit ratio."""
    import oracle  # test infrastructure: bench's cpu_baseline / --impl reference legs only

    host = host_cpu()
    core = min(os.sched_getaffinity(0))
    o = _oracle_sample(args, oracle, sample_requests, steps, core)
    o.update(cores=1, core=core, cpu_model=host["cpu_model"], nproc=host["nproc"],
             pinning=f"sched_setaffinity to core {core} (1 of {host['nproc']} cores) around the timed oracle calls")
    return o


class _Pinned:
    """the serial oracle runs pinned to one core (the input generation, torch on CPU, is not
    timed and keeps every core)"""

    def __init__(self, core):
        self.core = core

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {self.core})

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.saved)


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def _oracle_sample(args, oracle, sample_requests, steps, core):
    c = CONFIGS[args.config]
    Rs = sample_requests
    T = c["prompt"]
    need = Rs * c["Ly"] * c["H"] * ((T // c["Ch"]) + 4)
    cfg = oracle.make_config(R=Rs, Ly=c["Ly"], H=c["H"], d=c["d"], M=c["M"], W=c["W"], Ch=c["Ch"], Cl=c["Cl"],
                             P=int(need * 1.1), alpha_h=c["alpha_h"], alpha_l=c["alpha_l"])
    pool = oracle.OraclePool(cfg)
    wl = Workload(dict(c, R=Rs), 0, 1, torch.device("cpu"))
    sig, kk, vv = wl.prefill_inputs(T)
    sig_np = sig.numpy()
    k_np, v_np = kk.view(torch.int16).numpy().view(np.uint16), vv.view(torch.int16).numpy().view(np.uint16)
    with _Pinned(core):
        t0 = time.perf_counter()
        pool.classify_prefill(list(range(Rs)), [T] * Rs, sig_np, want_classes=False)
        pool.compact_alloc(None)
        t1 = time.perf_counter()
        pool.quant_write_prefill(k_np, v_np, sig_np)
        t2 = time.perf_counter()
    units = Rs * c["Ly"] * c["H"]
    # algorithmic bytes of the sample's bulk write (same accounting as the GPU)
    g = pool.geom
    geom = {k: dict(k_row=g[k].k_row, v_row=g[k].v_row) for k in (1, 2)}
    bb, _ = bulk_bytes_counts(int(pool.n_h.sum()), int(pool.n_l.sum()), units * (T - c["W"]), units * c["W"],
                              geom, c["d"])
    seq = np.full(Rs, T, np.int64)
    act = np.ones(Rs, bool)
    comp, cls, qw = [], [], []
    steps = steps or max(3, min(args.steps, 20))
    for s in range(steps):
        cand, nk, nv = wl.decode_inputs(seq, act)
        cand_np = cand.numpy()
        nk_np, nv_np = nk.view(torch.int16).numpy().view(np.uint16), nv.view(torch.int16).numpy().view(np.uint16)
        with _Pinned(core):
            a = time.perf_counter()
            st, dec = pool.classify_decode(cand_np)
            b = time.perf_counter()
            pool.compact_alloc(dec)
            cc = time.perf_counter()
            pool.quant_write_decode(dec, nk_np, nv_np, cand_np)
            dd = time.perf_counter()
        cls.append(b - a); comp.append(cc - b); qw.append(dd - cc)
        seq += 1
    scale = (c["R"] * c["Ly"] * c["H"]) / units
    return {
        "compact_us": statistics.mean(comp) * 1e6 * scale,
        "classify_us": statistics.mean(cls) * 1e6 * scale,
        "quant_us": statistics.mean(qw) * 1e6 * scale,
        "step_us": statistics.mean([a + b + q for a, b, q in zip(cls, comp, qw)]) * 1e6 * scale,
        "bulk_gbs": bb / (t2 - t1) / 1e9,
        "prefill_classify_s": t1 - t0,
        "sample": f"{Rs} of {c['R']} requests ({units} of {c['R'] * c['Ly'] * c['H']} units), prompt {T}, "
                  f"{steps} decode steps; µs scaled by the unit ratio x{scale:g}",
    }


def cpu_baseline_obj(o):
    return {"value": round(o["compact_us"], 3), "unit": "us", "cores": o["cores"], "kind": "oracle",
            "sample": o["sample"], "cpu_model": o["cpu_model"], "nproc": o["nproc"], "pinning": o["pinning"],
            "quant_write_gbs": round(o["bulk_gbs"], 3), "classify_us": round(o["classify_us"], 1),
            "quant_write_decode_us": round(o["quant_us"], 1), "step_us": round(o["step_us"], 1)}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    t0 = time.time()
    o = run_oracle_sample(args)
    c = CONFIGS[args.config]
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(o["compact_us"], 3),
        "unit": "us",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round((o["compact_us"] + o["classify_us"] + o["quant_us"]) / 1e3, 6),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp16 in / u8 codes (fp32 quantizer arithmetic)",
        "data": "synthetic (seeded counter-based, synth/)",
        "config": {"workload": f"{args.config} (oracle sample)", "global_batch": c["R"]},
        "cpu_baseline": cpu_baseline_obj(o),
        # the oracle's whole decode step, in our e2e unit (it runs on host buffers: no copies)
        "e2e": {"value": round(o["step_us"], 3), "unit": E2E_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.time() - t0, 1),
    }


def _spawned_rank(local, world, port, argv):
    """one rank of `bench.py --gpus N` started without torchrun: the torchrun environment, then main()"""
    os.environ.update(RANK=str(local), LOCAL_RANK=str(local), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.argv = [sys.argv[0]] + argv
    main()


def launch_ranks(args, argv):
    """`--gpus N` without WORLD_SIZE: spawn N ranks here, one per GPU (the same processes torchrun would start).
    Fails loudly when the node has fewer GPUs, unless --shared-device maps several ranks onto each GPU (a
    functional check of the N-rank path only: the ranks then share one GPU's SMs and HBM, and the counter
    all-reduce runs over gloo because NCCL refuses two ranks on one device)."""
    import socket

    import torch.multiprocessing as mp
    ndev = torch.cuda.device_count()
    if ndev < args.gpus and not args.shared_device:
        sys.exit(f"bench.py --gpus {args.gpus}: this node has {ndev} CUDA device(s); run on an {args.gpus}-GPU node "
                 f"(or pass --shared-device for a functional run of the {args.gpus}-rank path on fewer GPUs)")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mp.spawn(_spawned_rank, args=(args.gpus, port, argv), nprocs=args.gpus, join=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3_8b", choices=sorted(CONFIGS))
    ap.add_argument("--tile-units", type=int, default=0, help="compact_alloc scan tile (0 = library default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--next2", type=int, default=1, help="also time NEXT-2 decode steps (dkv_attend)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: fixed global batch (configs[1]'s 64 requests), heads sharded N-way")
    ap.add_argument("--shared-device", action="store_true",
                    help="allow more ranks than GPUs (functional check; counters over gloo)")
    argv = sys.argv[1:]
    args = ap.parse_args()
    assert args.warmup >= 3, "the driver's timing rules need >= 3 warm-up steps"
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(env_world or args.gpus)
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if env_world is None and args.gpus > 1:
        launch_ranks(args, argv)
        return
    if env_world is not None and int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
    rank, world, local = dist_init(args.shared_device)
    out = run_ours(args, rank, world, local)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_obj(run_oracle_sample(args))
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
