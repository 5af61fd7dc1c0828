"""NEXT-2 oracle pins: the normative exp (Q32) against the C library's exp; decode attention over the
compressed cache (Eq. 1, with GQA max) against an independent float64 numpy evaluation
that unpacks the page bytes itself; closed forms (identical keys -> uniform attention 1/n exactly; a
duplicated query head changes nothing); the running-mean significance update (Q33) against float64;
and a lifecycle in which classify / quant_write take t_c's significance from the window (cand_sig None)
with the invariants of PIN-10 after every call."""
import math

import numpy as np
import pytest

import oracle
from tests import harness as H


def test_exp_against_libm():
    xs = np.concatenate([np.linspace(-86.0, 0.0, 200001, dtype=np.float32),
                         -np.logspace(-8, 1.9, 5001).astype(np.float32), np.float32([0.0, -0.0])])
    lib = oracle.lib()
    got = np.array([lib.orc_exp(float(x)) for x in xs[::7]], np.float64)
    ref = np.exp(xs[::7].astype(np.float64))
    rel = np.abs(got - ref) / ref
    # bound of the algorithm (Q32): polynomial error + the rounding of t = x * log2(e), |t| * 2^-24 in the
    # exponent, i.e. about ln2 * 1.44 * |x| * 2^-24 = 6e-8 |x| relative
    bound = 5e-7 + 6.5e-8 * np.abs(xs[::7].astype(np.float64))   # + Horner rounding (~4 ulp)
    assert (rel <= bound).all(), (rel / bound).max()
    assert lib.orc_exp(0.0) == 1.0
    srt = np.sort(xs[::7])
    v = np.array([lib.orc_exp(float(x)) for x in srt])
    assert (np.diff(v) >= 0).all(), "exp must be monotone"


def _unpack(codes, bits, d):
    b = np.unpackbits(codes.astype(np.uint8), bitorder="little")
    vals = b.reshape(-1, bits) @ (1 << np.arange(bits))          # LSB-first per element (Q17)
    return vals[:d].astype(np.float64)


def _tokens64(pool, u):
    """(keys, values, positions) of unit u in Q31 order, dequantized in float64 from the page bytes"""
    c = pool.cfg
    d, L, W = c.d, pool.L, c.W
    ks, vs, ps = [], [], []
    for cls, n in ((1, pool.n_h[u]), (2, pool.n_l[u])):
        g = pool.geom[cls]
        for s in range(int(n)):
            pid = pool.table[u, s // g.C] if cls == 1 else pool.table[u, L - 1 - s // g.C]
            i = s % g.C
            pg = pool.pages[pid]
            for arr, off, row, meta, bits in ((ks, g.off_k, g.k_row, g.off_kmeta, g.kbits),
                                              (vs, g.off_v, g.v_row, g.off_vmeta, g.vbits)):
                sc, zc = pg[meta + 4 * i: meta + 4 * i + 4].view(np.float16).astype(np.float64)
                arr.append(sc * _unpack(pg[off + i * row: off + (i + 1) * row], bits, d) + zc)
            ps.append(int(pg[g.off_pos + 4 * i: g.off_pos + 4 * i + 4].view(np.int32)[0]))
    N = int(pool.seq_len[u // pool.LyH])
    for p in range(max(N - W, 0), N):
        ks.append(pool.win_k[u, p % W].view(np.float16).astype(np.float64))
        vs.append(pool.win_v[u, p % W].view(np.float16).astype(np.float64))
        ps.append(p)
    return np.array(ks), np.array(vs), np.array(ps)


def _pool_after_prefill(G=4, seed=3, mix=(0.35, 0.45, 0.20), R=2, lens=(150, 90)):
    scn = H.TINY.replace(R=R, Ly=2, H=2, d=64, M=256, W=16, P=2000, seed=seed, mix=mix, q_per_kv=G)
    o = H.OracleBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o], inp, life, list(range(R)), list(lens))
    return scn, o, inp, life


def test_attention_matches_float64_reference():
    scn, o, inp, life = _pool_after_prefill()
    p = o.pool
    G, d = 4, scn.d
    rng = np.random.default_rng(0)
    q = rng.normal(0, 1, size=(p.U, G, d)).astype(np.float16)
    sig_before = {u: _tokens64(p, u) for u in range(p.U)}
    st, out, probs = p.attend(q, want_out=True, want_probs=True)
    assert st == 0
    for u in range(p.U):
        k, v, pos = sig_before[u]
        logits = (q[u].astype(np.float64) @ k.T) / math.sqrt(d)      # Eq. 1
        a = np.exp(logits - logits.max(axis=1, keepdims=True))
        a /= a.sum(axis=1, keepdims=True)
        ref_out = a @ v
        assert np.allclose(out[u], ref_out, rtol=2e-4, atol=2e-5), u
        amax = a.max(axis=0)                                           # GQA: max over the group
        n = len(pos)
        assert np.allclose(probs[u, :n], amax, rtol=2e-5, atol=1e-7), u
        assert (probs[u, n:] == 0).all()


def test_identical_keys_give_uniform_attention_exactly():
    scn = H.TINY.replace(R=1, Ly=1, H=1, d=64, M=128, W=8, P=200, q_per_kv=2)
    o = H.OracleBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    sig, k, v = inp.prefill([0], [40])
    k = k * 0                                                          # every key dequantizes to 0
    assert o.classify_prefill([0], [40], sig) == 0 and o.compact_alloc(None) == 0
    assert o.quant_write_prefill(k, v, sig) == 0
    q = np.random.default_rng(1).normal(size=(1, 2, 64)).astype(np.float16)
    st, out, probs = o.pool.attend(q, want_out=False, want_probs=True)
    n = int(o.pool.n_h[0] + o.pool.n_l[0]) + 8
    assert (probs[0, :n] == np.float32(1.0) / np.float32(n)).all()


def test_duplicated_query_head_changes_nothing():
    _, o1, _, _ = _pool_after_prefill(G=1, seed=9)
    _, o2, _, _ = _pool_after_prefill(G=2, seed=9)
    q = np.random.default_rng(2).normal(size=(o1.pool.U, 1, 64)).astype(np.float16)
    _, out1, p1 = o1.pool.attend(q, want_probs=True)
    _, out2, p2 = o2.pool.attend(np.repeat(q, 2, axis=1), want_probs=True)
    assert np.array_equal(p1, p2) and np.array_equal(out2[:, 0], out1[:, 0]) and np.array_equal(out2[:, 1], out1[:, 0])


def test_significance_is_running_mean_of_later_scores():
    scn, o, inp, life = _pool_after_prefill(G=2, seed=4)
    p = o.pool
    rng = np.random.default_rng(5)
    u = 3
    k0, v0, pos0 = _tokens64(p, u)
    before = {}
    for cls, n in ((1, p.n_h[u]), (2, p.n_l[u])):
        for s in range(int(n)):
            rec = p.slot_record(cls, u, s)
            before[rec[5]] = np.uint32(rec[4]).view(np.float32)
    N = int(p.seq_len[u // p.LyH])
    q = rng.normal(size=(p.U, 2, 64)).astype(np.float16)
    _, _, probs = p.attend(q, want_out=False, want_probs=True)
    for cls, n in ((1, p.n_h[u]), (2, p.n_l[u])):
        for s in range(int(n)):
            rec = p.slot_record(cls, u, s)
            pos, new = rec[5], float(np.uint32(rec[4]).view(np.float32))
            i = int(np.nonzero(pos0 == pos)[0][0])
            c = N - 2 - pos                                            # later queries so far (Q33)
            ref = (float(before[pos]) * c + float(probs[u, i])) / (c + 1)
            assert abs(new - ref) <= 1e-6 * max(abs(ref), 1e-30), (pos, new, ref)


def test_lifecycle_with_window_significance():
    """classify / quant_write with cand_sig None read t_c's significance from the window; attention keeps it
    up to date; the pool invariants hold after every call."""
    scn = H.TINY.replace(R=3, Ly=2, H=2, d=64, M=200, W=8, P=3000, seed=12, q_per_kv=4, alpha_h=1.5, alpha_l=0.5)
    o = H.OracleBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o], inp, life, [0, 1, 2], [60, 33, 90])
    rng = np.random.default_rng(6)
    p = o.pool
    seen = set()
    for step in range(40):
        active = life.state == H.REQ_ACTIVE
        N = np.where(active, life.seq + 1, 0)
        _, k, v = inp.decode(N)
        st, dec = p.classify_decode(None)
        assert st == 0
        seen |= set(np.unique(dec["tc_class"]).tolist()) | {10 + x for x in np.unique(dec["v_action"]).tolist()}
        assert p.compact_alloc(dec) == 0 and p.quant_write_decode(dec, H._np(k), H._np(v), None) == 0
        life.seq[active] += 1
        q = rng.normal(size=(p.U, 4, 64)).astype(np.float16)
        assert p.attend(q, want_out=False)[0] == 0
        assert p.status == 0
        H.check_invariants(o.snapshot(), scn, o.L, o.geom)
    assert {1, 2, 11} <= seen and (12 in seen or 13 in seen), seen   # H, L, keep and a victim leaving


def test_eq1_helper_agrees_with_independent_unpacker():
    """tests/eq1.py (the float64 Eq. 1 the GPU attention is pinned to) against this file's own unpacker and
    float64 evaluation on an oracle pool: the same tokens, and the oracle's attention within the same bound."""
    from tests import eq1
    scn, o, inp, life = _pool_after_prefill(G=4, seed=5)
    p = o.pool
    geom = {c: dict(o.geom[c], kbits=p.geom[c].kbits, vbits=p.geom[c].vbits) for c in (1, 2)}
    snap = o.snapshot()
    q = np.random.default_rng(8).normal(0, 1, size=(p.U, 4, scn.d)).astype(np.float16)
    for u in range(p.U):
        k1, v1, p1 = _tokens64(p, u)
        k2, v2, p2 = eq1.unit_tokens64(snap["pages"], snap["table"][u], snap["n_h"][u], snap["n_l"][u],
                                       snap["seq_len"][u // p.LyH], snap["win_k"][u], snap["win_v"][u],
                                       geom, o.L, scn.W, scn.d)
        assert np.array_equal(k1, k2) and np.array_equal(v1, v2) and np.array_equal(p1, p2), u
    st, out, probs = p.attend(q, want_out=True, want_probs=True)
    assert st == 0
    eq1.check_units(snap, geom, o.L, scn.W, scn.d, p.LyH, q, out, probs, range(p.U), where="oracle")
