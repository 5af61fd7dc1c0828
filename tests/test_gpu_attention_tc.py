"""NEXT-2 on tensor cores (dkv_attend_tc) pinned to the paper's formula directly: the attention outputs and the
per-token scores (max over the GQA group) against Eq. 1 evaluated in float64 from the GPU
pool's own page bytes (tests/eq1.py), the significance it writes back against the float64 running mean of the
float64 scores (Q33) tracked over the whole lifecycle, the section minima against the values it wrote
(exact), and — downstream — every victim the next dkv_classify takes from those minima is, in float64, the
section minimum within the tolerance (margin-aware: ties closer than the tolerance may go either way)."""
import numpy as np
import pytest
import torch

from tests import eq1
from tests import harness as H

pytestmark = pytest.mark.gpu

SIG_RTOL = 1e-4          # written significance vs the float64 running mean (errors of ~1e-6 per step, averaged)


def _sig_map(snap, geom, L, W, u, LyH):
    """{position: (class, slot, significance)} of unit u's stored tokens + {position: sig} of its window"""
    out = {}
    for cls, n in ((1, int(snap["n_h"][u])), (2, int(snap["n_l"][u]))):
        g = geom[cls]
        for s in range(n):
            k = s // g["C"] if cls == 1 else L - 1 - s // g["C"]
            pg = snap["pages"][snap["table"][u, k]]
            i = s % g["C"]
            pos = int(pg[g["off_pos"] + 4 * i: g["off_pos"] + 4 * i + 4].view(np.int32)[0])
            sg = float(pg[g["off_score"] + 4 * i: g["off_score"] + 4 * i + 4].view(np.float32)[0])
            out[pos] = (cls, s, sg)
    N = int(snap["seq_len"][u // LyH])
    for pos in range(max(N - W, 0), N):
        out[pos] = (0, -1, float(snap["win_sig"][u, pos % W]))
    return out


def _run(scn, lens, steps, seed=0, frees=()):
    from tests.gpu_backend import GpuBackend, dec_np
    g = GpuBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    rng = np.random.default_rng(seed)
    G, d, W, L = scn.q_per_kv, scn.d, scn.W, g.L
    H.admit([g], inp, life, list(range(len(lens))), lens)
    sig64 = {}                                                  # (u, pos) -> float64 significance
    snap = g.snapshot()
    for u in range(scn.U):
        for pos, (_, _, sg) in _sig_map(snap, g.geom, L, W, u, scn.LyH).items():
            sig64[(u, pos)] = sg
    frees = dict(frees)
    worst = 0.0
    for step in range(steps + 1):
        if step > 0:                                            # a decode step driven by the written significance
            active = life.state == H.REQ_ACTIVE
            N = np.where(active, life.seq + 1, 0)
            _, k, v = inp.decode(N)
            before = g.snapshot()
            _, dg = g.classify_decode(None)
            dec = dec_np(dg).copy()
            # margin-aware victim check: the victim is the float64 section minimum within the tolerance
            for u in range(scn.U):
                if dec["v_action"][u] not in (2, 3):
                    continue
                cls = 1 if dec["tc_class"][u] == 1 else 2
                m = _sig_map(before, g.geom, L, W, u, scn.LyH)
                sec = {pos: sig64[(u, pos)] for pos, (c, _, _) in m.items() if c == cls}
                vpos = [pos for pos, (c, s, _) in m.items() if c == cls and s == dec["v_slot"][u]][0]
                lo = min(sec.values())
                assert sec[vpos] <= lo * (1 + 2 * SIG_RTOL) + 1e-12, (step, u, sec[vpos], lo)
            assert g.compact_alloc(dg) == 0 and g.quant_write_decode(dg, k, v, None) == 0
            for u in range(scn.U):                              # t_c leaves the window; the new token enters at 0
                r = u // scn.LyH
                if active[r]:
                    sig64[(u, int(N[r]) - 1)] = 0.0
            life.seq[active] += 1
            if step in frees:
                H.free([g], life, frees[step])
                for uu in [x for x in list(sig64) if x[0] // scn.LyH in frees[step]]:
                    del sig64[uu]
        q = rng.normal(0, 1, size=(scn.U, G, d)).astype(np.float16)
        snap = g.snapshot()
        _, og, pg = g.attend_tc(q, want_out=True, want_probs=True)
        live = [u for u in range(scn.U) if snap["req_state"][u // scn.LyH] == H.REQ_ACTIVE]
        eq1.check_units(snap, g.geom, L, W, d, scn.LyH, q, og, pg, live, where=f"tc step {step}")
        after = g.snapshot()
        for u in range(scn.U):
            r = u // scn.LyH
            if after["req_state"][r] != H.REQ_ACTIVE:
                continue
            kk, vv, pos = eq1.unit_tokens64(snap["pages"], snap["table"][u], snap["n_h"][u], snap["n_l"][u],
                                            snap["seq_len"][r], snap["win_k"][u], snap["win_v"][u], g.geom, L, W, d)
            _, a = eq1.attend64(q[u], kk, vv)
            N = int(snap["seq_len"][r])
            m = _sig_map(after, g.geom, L, W, u, scn.LyH)
            for i, ps in enumerate(pos):
                c = N - 2 - int(ps)
                key = (u, int(ps))
                if c >= 0:
                    sig64[key] = (sig64.get(key, 0.0) * c + float(a[i])) / (c + 1)
                got = m[int(ps)][2]
                ref = sig64.get(key, 0.0)
                err = abs(got - ref) / max(abs(ref), 1e-6)
                worst = max(worst, err)
                assert err <= SIG_RTOL, (step, u, ps, got, ref)
            # the section minima: exact argmin of the values written
            sm = after_secmin = g.pool.views()["secmin"][u].cpu().numpy()
            for ci, cls in enumerate((1, 2)):
                keys = [(np.float32(sg).view(np.uint32), ps, s) for ps, (c, s, sg) in m.items() if c == cls]
                if keys:
                    b = min(keys, key=lambda x: (int(x[0]), x[1]))
                    assert (int(sm[3 * ci]) & 0xFFFFFFFF, int(sm[3 * ci + 1]), int(sm[3 * ci + 2])) == \
                           (int(b[0]), int(b[1]), int(b[2])), (step, u, cls)
            assert int(sm[6]) == 1
    st, _ = g.pool.query()
    assert st == 0
    return worst


@pytest.mark.parametrize("G", [1, 4, 5, 8])
def test_attention_tc_d128_multi_page(G):
    scn = H.TINY.replace(R=3, Ly=2, H=3, d=128, M=700, W=64, P=6000, seed=21, q_per_kv=G, alpha_h=1.0, alpha_l=0.02)
    _run(scn, [520, 70, 300], steps=8, seed=G, frees=[(4, [1])])


@pytest.mark.parametrize("G", [2, 7])
def test_attention_tc_d64_ragged(G):
    scn = H.TINY.replace(R=4, Ly=2, H=2, d=64, M=900, W=16, P=6000, seed=31 + G, q_per_kv=G, alpha_h=1.0,
                         alpha_l=0.02)
    _run(scn, [700, 9, 130, 16], steps=6, seed=G)


def test_attention_tc_qwen_thresholds_no_pruning():
    # alpha (3, 0) as in the Qwen thinking config: nothing pruned, low sections full of ties at exact zero
    scn = H.TINY.replace(R=2, Ly=2, H=2, d=128, M=2000, W=64, P=6000, seed=13, q_per_kv=5, alpha_h=3.0,
                         alpha_l=0.0, mix=(0.4, 0.6, 0.0))
    _run(scn, [1500, 600], steps=5, seed=7)


def test_attention_tc_long_context():
    """30k-token contexts, G = 8 (the Qwen thinking shape's length): logits live in the CTA's scratch slot, not in
    shared memory — outputs and scores against Eq. 1 in float64, as for the short contexts"""
    from tests.gpu_backend import GpuBackend
    scn = H.TINY.replace(R=1, Ly=1, H=2, d=128, M=33792, W=64, P=4000, seed=13, q_per_kv=8, alpha_h=3.0,
                         alpha_l=0.0, mix=(0.4, 0.6, 0.0))
    g = GpuBackend(scn)
    H.admit([g], H.Inputs(scn), H.Lifecycle(scn), [0], [30000])
    q = np.random.default_rng(1).normal(size=(scn.U, 8, 128)).astype(np.float16)
    snap = g.snapshot()
    _, og, pg = g.attend_tc(q, want_out=True, want_probs=True)
    eq1.check_units(snap, g.geom, g.L, scn.W, scn.d, scn.LyH, q, og, pg, list(range(scn.U)), where="tc 30k")


@pytest.mark.parametrize("W", [0, 24])
def test_attention_tc_window_not_a_chunk_multiple(W):
    """A window ring of W = 24 slots (one full and one partial 16-slot MMA chunk; contexts shorter than W leave slots
    empty) and no window at all (W = 0: t_c is the new token), against Eq. 1 in float64 over a lifecycle"""
    scn = H.TINY.replace(R=3, Ly=2, H=2, d=128, M=600, W=W, P=6000, seed=41 + W, q_per_kv=4, alpha_h=1.0,
                         alpha_l=0.02)
    _run(scn, [300, 11, 90], steps=5, seed=W)


@pytest.mark.parametrize("G,W", [(4, 64), (8, 24), (5, 0)])
def test_attention_tc_split_sequence(G, W):
    """Few active units with long contexts take the split-sequence form: each unit's pages split over
    several CTAs whose partial softmax states a merge kernel combines (it also runs the significance pass) — outputs,
    scores, the written significance and the section minima against Eq. 1 in float64 over a lifecycle, as for the
    single-CTA form"""
    scn = H.TINY.replace(R=2, Ly=1, H=2, d=128, M=5000, W=W, P=8000, seed=51 + G, q_per_kv=G, alpha_h=1.0,
                         alpha_l=0.02)
    _run(scn, [3000, 2300], steps=4, seed=G, frees=[(2, [1])])
