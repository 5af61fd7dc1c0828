"""NEXT-4 on the GPU: the three-level tier FP16-K8V4-K4V2 (readings Q38-Q44) bit-exact with the
oracle after every call — decisions, ring, pointers, both tables (the unidirectional TOP table and the
bidirectional one), counts, window and page bytes — through prefill, decode steps with significance drift (TOP
pages included), TOP victims moving down (Q39/Q42), frees recycled by the decode fast path (deferred copies) and
by the barrier path (a tight pool), re-admission, multi-tile scans, a decode-step CUDA graph, and a non-finite
TOP token (Q30)."""
import numpy as np
import pytest
import torch

import oracle
from tests import harness as H
from tests.test_gpu_parity import _lifecycle

pytestmark = pytest.mark.gpu


def test_top_tier_tiny_every_call():
    scn = H.TINY.replace(R=4, Ly=2, H=4, d=64, M=256, W=16, P=4000, seed=61, top_tier=1, alpha_t=2.0, Ct=4)
    o, g, life = _lifecycle(scn, steps=40, prompt_lens=[64, 100, 33, 150], frees=[(12, [1]), (20, [0, 3])],
                            readmit_len=90)
    assert (o.pool.n_t > 0).any()


@pytest.mark.parametrize("tile_units,tight", [(256, False), (1024, True)])
def test_top_tier_d128_victims_and_recycling(tile_units, tight):
    # alpha / n prompt thresholds keep stored TOP significance near alpha_t / N, so drift moves TOP victims down
    base = H.TINY.replace(R=6, Ly=4, H=8, d=128, M=700, W=64, P=60000, seed=62, top_tier=1, alpha_t=1.5,
                          alpha_h=1.0, alpha_l=0.2, Ct=8, prompt_denominator=1, tile_units=tile_units)
    lens = [300, 150, 520, 64, 200, 90]
    scn = base
    if tight:                                                    # free < U: the barrier path recycles in place
        probe = H.OracleBackend(base)
        inp, life = H.Inputs(base), H.Lifecycle(base)
        H.admit([probe], inp, life, list(range(6)), lens)
        scn = base.replace(P=(60000 - int(probe.pool.free)) + 3 * base.U // 4)   # OOM-free, free < U
    o, g, life = _lifecycle(scn, steps=24, prompt_lens=lens, frees=[(6, [2]), (14, [0, 4])], readmit_len=260,
                            pages_every=3)
    assert (o.pool.n_t > 0).any()


def test_top_tier_graph_replay():
    from tests.gpu_backend import GpuBackend, compare_state, dec_np
    from paper_2412_03131_b200 import dkv as D
    scn = H.TINY.replace(R=5, Ly=2, H=4, d=64, M=300, W=16, P=6000, seed=63, top_tier=1, alpha_t=2.0, Ct=4,
                         tile_units=256)
    o, g = H.OracleBackend(scn), GpuBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, list(range(scn.R)), [70, 120, 40, 90, 64])
    dev = g.device
    sig = torch.zeros(scn.U, dtype=torch.float32, device=dev)
    k = torch.zeros((scn.U, scn.d), dtype=torch.int16, device=dev)
    v = torch.zeros_like(k)
    dec = g.pool.new_decisions()
    graph = g.pool.decode_graph(1, sig, k, v, dec, D.DKV_GRAPH_PDL)
    for step in range(20):
        o.drift(step)
        g.drift(step)
        active = life.state == H.REQ_ACTIVE
        N = np.where(active, life.seq + 1, 0)
        cand, kk, vv = inp.decode(N)
        st, do = o.classify_decode(cand)
        assert st == 0 and o.compact_alloc(do) == 0 and o.quant_write_decode(do, kk, vv, cand) == 0
        sig.copy_(cand.to(dev))
        k.copy_(kk.to(dev).view(torch.int16))
        v.copy_(vv.to(dev).view(torch.int16))
        graph.launch()
        torch.cuda.synchronize()
        life.seq[active] += 1
        assert np.array_equal(dec_np(do).view(np.uint8), dec_np(dec).view(np.uint8)), step
        compare_state(o.snapshot(), g.snapshot(), where=f"graph step {step}")
        if step == 7:
            H.free([o, g], life, [1, 3])                          # TOP pages recycled inside the next replay
    graph.close()


def test_top_tier_nonfinite_top_token_rejected():
    from tests.gpu_backend import GpuBackend, compare_state
    scn = H.TINY.replace(R=2, Ly=2, H=2, d=64, M=200, W=16, P=2000, seed=64, top_tier=1, alpha_t=2.0, Ct=4)
    o, g = H.OracleBackend(scn), GpuBackend(scn)
    inp = H.Inputs(scn)
    sig, k, v = inp.prefill([0, 1], [80, 80])
    # a TOP token of unit 0 (significance at or above alpha_t / (t + 1)) gets a NaN key element
    s0 = sig[0, 0].numpy()
    t_top = int(np.nonzero(s0[:64] >= np.float32(2.0) / (np.arange(64) + 1).astype(np.float32))[0][3])
    k = k.clone()
    k.view(torch.int16)[0, 0, t_top, 5] = 0x7E00
    for b in (o, g):
        assert b.classify_prefill([0, 1], [80, 80], sig) == 0
        assert b.compact_alloc(None) == 0
        assert b.quant_write_prefill(k, v, sig) == 0
    assert o.pool.status == oracle.ERR_NONFINITE
    compare_state(o.snapshot(), g.snapshot(), where="nonfinite TOP token")
    assert g.take_status() == oracle.ERR_NONFINITE


def test_top_tier_rejects_attention_and_bad_thresholds():
    from tests.gpu_backend import GpuBackend
    from paper_2412_03131_b200 import dkv as D
    scn = H.TINY.replace(R=2, Ly=1, H=2, d=64, M=128, W=16, P=500, top_tier=1, alpha_t=2.0, Ct=4, q_per_kv=2)
    g = GpuBackend(scn)
    q = np.zeros((scn.U, 2, 64), np.float16)
    with pytest.raises(RuntimeError):
        g.attend(q)
    with pytest.raises(RuntimeError):
        g.attend_tc(q)
    with pytest.raises(RuntimeError):                             # per-head alpha_h above alpha_t (Q38)
        g.set_head_thresholds(np.full(2, 3.0, np.float32), np.zeros(2, np.float32))
    for bad in (dict(alpha_t=0.5), dict(prefill_workflow=1), dict(Ct=6)):
        s2 = scn.replace(**bad)
        cfg = D.make_config(s2.R, s2.Ly, s2.H, s2.d, s2.M, s2.W, s2.Ch, s2.Cl, P=s2.P, alpha_h=s2.alpha_h,
                            alpha_l=s2.alpha_l, prefill_workflow=s2.prefill_workflow, top_tier=1, alpha_t=s2.alpha_t,
                            page_tokens_top=s2.Ct)
        assert D.dkv_arena_bytes(cfg) == 0
