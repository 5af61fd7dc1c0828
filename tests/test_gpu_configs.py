"""GPU-vs-oracle parity on the shapes of BASELINE.json's other configs, scaled so the oracle runs in seconds
(every call compared bit-exactly: decisions, ring, pointers, tables, counts, request state, window, pages):

  configs[2] Qwen-32B-style thinking shard — 64-layer model, 8 KV heads sharded 4-way (this pool holds heads
             2-3), alpha = (3, 0) so nothing is pruned (Q24), max_seq_len 33792 (table length 2113) and
             requests at very different progress (long sections: the classify scan runs many batches);
  configs[3] Llama-3-70B shard — 8-way head sharding (one KV head per pool, global head 5), 7168-token
             prompts, max_seq_len 9216, alpha = (1, 0);
  configs[4] fragmentation stress — many requests with random prompt lengths, random finish order and
             admission that keeps the pool about 90 % occupied, for hundreds of steps (ring wraparound,
             recycling every few steps, interleaved prefill and decode), both prompt workflows.
The full-size configs are exercised by bench.py (--config); their per-unit arithmetic is identical."""
import numpy as np
import pytest

import oracle
from tests import harness as H

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _pair(scn):
    from tests.gpu_backend import GpuBackend
    return H.OracleBackend(scn), GpuBackend(scn)


def _check(o, g, where, decs=None, pages=True):
    from tests.gpu_backend import compare_state, dec_np
    if decs is not None:
        a, b = dec_np(decs[0]), dec_np(decs[1])
        if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
            bad = np.nonzero(a != b)[0]
            raise AssertionError(f"[{where}] decisions differ at units {bad[:8].tolist()}")
    so, sg = o.snapshot(pages=pages), g.snapshot(pages=pages)
    compare_state(so, sg, where=where)
    assert sg["status"] == 0 and o.pool.status == 0, where


def test_qwen32b_thinking_shard_long_sections():
    scn = H.Scenario(R=3, Ly=4, H=2, H_total=8, h0=2, d=128, M=33792, W=64, Ch=16, Cl=32, P=20000,
                     alpha_h=3.0, alpha_l=0.0, mix=(0.40, 0.60, 0.0), seed=3)
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [0, 1, 2], [21000, 700, 9000])
    _check(o, g, "prefill")
    for step in range(12):
        decs = H.decode_step([o, g], inp, life, step)
        _check(o, g, f"step {step}", decs, pages=step % 4 == 0)
        if step == 5:
            H.free([o, g], life, [1])
    H.admit([o, g], inp, life, [1], [15000])                 # re-admitted after its pages were recycled
    _check(o, g, "re-admission")
    for step in range(12, 16):
        decs = H.decode_step([o, g], inp, life, step)
        _check(o, g, f"step {step}", decs, pages=step == 15)


def test_llama70b_one_head_shard():
    scn = H.Scenario(R=2, Ly=16, H=1, H_total=8, h0=5, d=128, M=9216, W=64, Ch=16, Cl=32, P=16000,
                     alpha_h=1.0, alpha_l=0.0, mix=(0.25, 0.75, 0.0), seed=4)
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [0, 1], [7168, 7168])
    _check(o, g, "prefill")
    for step in range(16):
        decs = H.decode_step([o, g], inp, life, step)
        _check(o, g, f"step {step}", decs, pages=step % 5 == 0)


@pytest.mark.parametrize("workflow", [0, 1])
def test_fragmentation_stress(workflow):
    rng = np.random.default_rng(5 + workflow)
    scn = H.Scenario(R=40, Ly=2, H=2, d=64, M=1536, W=16, Ch=16, Cl=32, P=4400, alpha_h=1.0, alpha_l=0.02,
                     seed=5, prefill_workflow=workflow)
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    target = int(0.9 * scn.P)
    gen_left = np.zeros(scn.R, np.int64)
    LyH = scn.LyH
    recycled = admitted = 0

    def used():
        return scn.P - o.pool.free

    def admit_until_full():
        nonlocal admitted
        idle = [r for r in range(scn.R) if life.state[r] == H.REQ_IDLE]
        rng.shuffle(idle)
        for r in idle:
            T = int(rng.integers(16, 1024))
            worst = LyH * (-(-max(T - scn.W, 0) // scn.Ch) + 1)      # conservative block (+ top-up) per unit
            if used() + worst + LyH * 4 > target:
                break
            H.admit([o, g], inp, life, [r], [T])
            gen_left[r] = int(rng.integers(8, 400))
            gen_left[r] = min(gen_left[r], scn.M - T)
            admitted += 1

    admit_until_full()
    _check(o, g, "initial admissions")
    def settle():                                               # a decode step recycled the freed requests
        life.state[life.state == H.REQ_PENDING_FREE] = H.REQ_IDLE

    for step in range(600):
        decs = H.decode_step([o, g], inp, life, step)
        settle()
        act = life.state == H.REQ_ACTIVE
        gen_left[act] -= 1
        _check(o, g, f"step {step}", decs, pages=step % 20 == 0)
        if step % 50 == 0:                                      # the device audit agrees (dkv_audit)
            a = g.pool.audit()
            assert a["used_pages"] + a["free_pages"] == scn.P and a["used_pages"] == scn.P - o.pool.free, (step, a)
            assert all(v == 0 for k, v in a.items() if k not in ("used_pages", "free_pages")), (step, a)
        done = [r for r in range(scn.R) if life.state[r] == H.REQ_ACTIVE and gen_left[r] <= 0]
        rng.shuffle(done)
        if done:
            H.free([o, g], life, done)                          # random finish order
            recycled += len(done)
        if step % 3 == 2:
            H.decode_step([o, g], inp, life, 10_000 + step)      # recycles PENDING_FREE requests
            settle()
            act = life.state == H.REQ_ACTIVE
            gen_left[act] -= 1
            admit_until_full()
            _check(o, g, f"churn {step}", pages=False)
    assert recycled > 20 and admitted > 40, (recycled, admitted)
    _check(o, g, "end")
