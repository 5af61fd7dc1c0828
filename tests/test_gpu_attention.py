"""NEXT-2 GPU-vs-oracle parity through the C ABI: decode attention over the compressed cache (dkv_attend),
the running-mean significance it writes back (page score segments, window significance), and decode steps
whose classify / quant_write take t_c's significance from the window (d_sig NULL) with the victim taken
from the section minima recorded by the attention kernel — bit-exact outputs, per-token scores, decisions
and pool state after every call (readings Q31-Q34)."""
import numpy as np
import pytest
import torch

from tests import eq1
from tests import harness as H

pytestmark = pytest.mark.gpu


def _run(scn, lens, steps, frees=(), readmit=None, seed=0):
    from tests.gpu_backend import GpuBackend, compare_state, dec_np
    o, g = H.OracleBackend(scn), GpuBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    rng = np.random.default_rng(seed)
    G, d = scn.q_per_kv, scn.d

    def same(where, pages=True):
        compare_state(o.snapshot(pages=pages), g.snapshot(pages=pages), where=where)

    def attend(where):
        q = rng.normal(0, 1, size=(scn.U, G, d)).astype(np.float16)
        _, oo, po = o.attend(q, want_out=True, want_probs=True)
        _, og, pg = g.attend(q, want_out=True, want_probs=True)
        assert np.array_equal(po.view(np.uint32), pg.view(np.uint32)), f"[{where}] per-token scores differ"
        assert np.array_equal(oo.view(np.uint32), og.view(np.uint32)), f"[{where}] attention outputs differ"
        # the GPU result pinned to the paper's formula itself: Eq. 1 in float64 from the GPU pool's page bytes
        sg = g.snapshot()
        units = range(scn.U) if scn.U * scn.M <= 200000 else range(0, scn.U, max(1, scn.U // 16))
        eq1.check_units(sg, g.geom, g.L, scn.W, d, scn.LyH, q, og, pg, units, where=where)
        same(where + " attend")

    H.admit([o, g], inp, life, list(range(len(lens))), lens)
    same("prefill")
    attend("prefill")
    pending = {}
    frees = dict(frees)
    for step in range(steps):
        active = life.state == H.REQ_ACTIVE
        N = np.where(active, life.seq + 1, 0)
        _, k, v = inp.decode(N)
        (_, do), (_, dg) = o.classify_decode(None), g.classify_decode(None)
        a, b = dec_np(do), dec_np(dg)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"decisions differ at step {step}"
        assert o.compact_alloc(do) == 0 and g.compact_alloc(dg) == 0
        assert o.quant_write_decode(do, k, v, None) == 0 and g.quant_write_decode(dg, k, v, None) == 0
        life.seq[active] += 1
        same(f"step {step}", pages=step % 3 == 0)
        attend(f"step {step}")
        assert o.pool.status == 0
        for r, t in list(pending.items()):
            if step >= t:
                H.admit([o, g], inp, life, [r], [readmit])
                same(f"re-admit {r}")
                del pending[r]
        if step in frees:
            H.free([o, g], life, frees[step])
            for r in frees[step]:
                pending[r] = step + 2
    return o, g


def test_attention_parity_tiny():
    scn = H.TINY.replace(q_per_kv=4, M=160)
    _run(scn, [64, 64, 64, 64], steps=30, frees=[(10, [2])], readmit=40)


@pytest.mark.parametrize("G", [1, 2, 4, 5, 7, 8])
def test_attention_parity_multi_page_d128(G):
    # d = 128, K8V4 / K4V2, several pages per section, ragged prompts, GQA groups of 1 / 5 / 8 heads
    scn = H.TINY.replace(R=3, Ly=2, H=3, d=128, M=700, W=64, P=6000, seed=21, q_per_kv=G,
                         alpha_h=1.0, alpha_l=0.02)
    _run(scn, [520, 70, 300], steps=12, frees=[(4, [1])], readmit=200, seed=G)


@pytest.mark.parametrize("G", [2, 7])
def test_attention_parity_d64_ragged_windows(G):
    # d = 64 (half-width pages), K8V4 / K4V2, a 16-token window (one window page) next to prompts shorter than
    # the window, ragged multi-page sections, frees and re-admission
    scn = H.TINY.replace(R=4, Ly=2, H=2, d=64, M=900, W=16, P=6000, seed=31 + G, q_per_kv=G,
                         alpha_h=1.0, alpha_l=0.02)
    _run(scn, [700, 9, 130, 16], steps=10, frees=[(3, [0])], readmit=333, seed=G)


def test_fused_victim_matches_scan():
    """The classify fast path (section minima written by dkv_attend) and the scan give the same decisions:
    two pools with the same history, one with its minima invalidated."""
    from tests.gpu_backend import GpuBackend, dec_np
    scn = H.TINY.replace(R=3, Ly=2, H=4, d=64, M=300, W=16, P=4000, seed=8, q_per_kv=2)
    rng = np.random.default_rng(3)
    q = rng.normal(size=(scn.U, 2, 64)).astype(np.float16)
    decs = []
    for invalidate in (False, True):
        g = GpuBackend(scn)
        inp, life = H.Inputs(scn), H.Lifecycle(scn)
        H.admit([g], inp, life, [0, 1, 2], [200, 120, 64])
        g.attend(q, want_out=False)
        v = g.pool.views()
        assert (v["secmin"][:, 6].cpu() == 1).all()
        if invalidate:
            v["secmin"][:, 6] = 0                                # force the scan
            torch.cuda.synchronize()
        _, d = g.classify_decode(None)
        decs.append(dec_np(d).copy())
    assert np.array_equal(decs[0].view(np.uint8), decs[1].view(np.uint8))


def test_attention_parity_long_context():
    # Qwen-32B-style thinking shard (BASELINE configs[2] shape): 33k max length, GQA group of 5, alpha (3, 0):
    # the logits of a 20k-token request do not fit in shared memory -> the persistent form with HBM slots
    scn = H.TINY.replace(R=2, Ly=2, H=2, d=128, M=33792, W=64, P=8000, seed=13, q_per_kv=5,
                         alpha_h=3.0, alpha_l=0.0, mix=(0.4, 0.6, 0.0))
    _run(scn, [20000, 6000], steps=3, seed=7)
