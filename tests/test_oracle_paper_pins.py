"""Pins taken from the paper's own worked examples and arithmetic (fixtures in tests/golden/, each with its
citation): Fig. 5 replay (PIN-1), Fig. 1 payload accounting (PIN-2), the 32 MB table figure (PIN-3), the
table-length bound (PIN-12), and the page contents written by the prompt path."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests import harness as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_fig5_replay():
    g = _load("fig5.json")
    c = g["config"]
    pool = oracle.OraclePool(oracle.make_config(**c))
    pool.start, pool.free = g["initial"]["start"], g["initial"]["free"]    # pages 0-4 in use before
    n = g["prompt_len"]
    sig = np.array(g["sig"], np.float32).reshape(1, 2, n)
    st, reclaimed = pool.prefill_conservative([0], [n], sig)
    assert st == oracle.OK and pool.status == oracle.OK
    e = g["expect"]
    L = pool.L
    for head, u in (("A", 0), ("B", 1)):
        row = pool.table[u]
        hi = list(row[:len(e["high_pages"][head])])
        lo = [int(row[L - 1 - k]) for k in range(len(e["low_pages"][head]))]
        assert hi == e["high_pages"][head] and lo == e["low_pages"][head]
        assert sorted(int(x) for x in row if x >= 0) == sorted(e["high_pages"][head] + e["low_pages"][head])
    assert list(reclaimed) == e["reclaimed_in_order"]
    assert list(pool.ring[:3]) == e["ring_head_after"]
    assert pool.start == e["start_after"] and pool.free == e["free_after"]
    P = c["P"]
    free_region = [int(pool.ring[(pool.start + i) % P]) for i in range(pool.free)]
    assert free_region == e["free_region_after"]


def test_fig1_payload_accounting():
    g = _load("fig1.json")
    d = 64
    pool = oracle.OraclePool(oracle.make_config(R=1, Ly=1, H=2, d=d, M=8, W=0, Ch=2, Cl=4, P=64))
    val = {"H": 2.0, "L": 0.05, "P": 0.001}    # H >= 1/i; 0.02/i <= L < 1/i; P < 0.02/i for i <= 5
    sig = np.array([[val[x] for x in g["head_A"]], [val[x] for x in g["head_B"]]], np.float32).reshape(1, 2, 5)
    st, cls = pool.classify_prefill([0], [5], sig)
    assert st == 0
    assert pool.compact_alloc(None) == 0
    k = np.zeros((1, 2, 5, d), np.float16)
    assert pool.quant_write_prefill(k, k, sig) == 0
    gh, gl = pool.geom[oracle.CLS_HIGH], pool.geom[oracle.CLS_LOW]
    fp16 = 5 * d * 2
    frac = {}
    for name, u in (("A", 0), ("B", 1)):
        frac[name + "_keys"] = Fraction(int(pool.n_h[u]) * gh.k_row + int(pool.n_l[u]) * gl.k_row, fp16)
        frac[name + "_values"] = Fraction(int(pool.n_h[u]) * gh.v_row + int(pool.n_l[u]) * gl.v_row, fp16)
    e = g["expect"]
    for key in ("A_keys", "A_values", "B_keys", "B_values"):
        assert frac[key] == Fraction(e[key]).limit_denominator(1000), key
    avg = sum(frac.values()) / 4
    assert avg == Fraction(33, 160) and float(avg) == e["average"]
    assert f"{100 * float(avg):.1f}%" == e["average_printed"]


def test_table_bytes_32MiB():
    # batch 128, Llama-3-8B (32 layers, 8 KV heads) -> "only 32 MB"; 8192-token requests (1 GB of
    # FP16 KV each at 128 KiB/token) with 32 tokens per high page give the paper's L = 256.
    cfg = oracle.make_config(R=128, Ly=32, H=8, d=128, M=8192, W=64, Ch=32, Cl=64, P=1)
    geo = oracle.geometry(cfg)
    assert geo["L"] == 256
    assert oracle.table_bytes(128, 32, 8, geo["L"]) == 32 * 2 ** 20
    assert 32 * 8 * 128 * 2 * 2 * 8192 == 2 ** 30                         # "a single request occupies 1 GB"


def test_table_length_never_overflows_small_geometries():
    # PIN-12 (Q12): pages needed = ceil(a/Ch) + ceil(b/Cl) for a + b <= M - W stored tokens must fit L.
    for Ch in range(1, 5):
        for Cl in range(Ch, 3 * Ch + 1):
            for W in range(0, 6):
                for M in range(1, 25):
                    L = oracle.geometry(oracle.make_config(M=M, W=W, Ch=Ch, Cl=Cl, P=1))["L"]
                    worst = max(-(-a // Ch) + -(-b // Cl) for a in range(0, M + 1) for b in range(0, M - a + 1)
                                if a + b <= max(M - W, 0))
                    assert worst <= L, (Ch, Cl, W, M)
    # and the paper's unmodified rule L = M / C_h does overflow without a window (the reason for Q12)
    assert -(-1 // 2) + -(-1 // 2) > 2 // 2


def test_prefill_page_contents():
    """Each kept token lands in slot = its rank among same-class tokens (position order), with codes =
    quantize(its K/V) at the class bits, meta = (s16, z16), score = its significance, pos = its index."""
    scn = H.TINY
    o = H.OracleBackend(scn)
    inp = H.Inputs(scn)
    life = H.Lifecycle(scn)
    sig = H.admit([o], inp, life, [0, 2], [64, 50])
    _, k, v = inp.prefill([0, 2], [64, 50])
    sg, kk, vv = H._np(sig), H._np(k), H._np(v)
    p = o.pool
    for i, (r, n) in enumerate(((0, 64), (2, 50))):
        for j in range(scn.LyH):
            u = r * scn.LyH + j
            rank = {1: 0, 2: 0}
            for t in range(n - scn.W):
                s = np.float32(sg[i, j, t]) + np.float32(0)
                th, tl = np.float32(scn.alpha_h) / np.float32(t + 1), np.float32(scn.alpha_l) / np.float32(t + 1)
                cls = 1 if s >= th else 2 if s >= tl else 3
                if cls == 3:
                    continue
                slot = rank[cls]
                rank[cls] += 1
                kc, km, vc, vm, sgb, ps = p.slot_record(cls, u, slot)
                gm = p.geom[cls]
                _, ck, sk, zk = oracle.quantize(kk[i, j, t].view(np.float16).astype(np.float32), gm.kbits)
                _, cv, sv, zv = oracle.quantize(vv[i, j, t].view(np.float16).astype(np.float32), gm.vbits)
                assert np.array_equal(kc, ck) and np.array_equal(vc, cv)
                assert km == sk | (zk << 16) and vm == sv | (zv << 16)
                assert sgb == int(np.float32(s).view(np.uint32)) and ps == t
            assert rank[1] == p.n_h[u] and rank[2] == p.n_l[u]
            # window: the newest W tokens at slot pos mod W, bit-exact fp16
            for t in range(max(n - scn.W, 0), n):
                assert np.array_equal(p.win_k[u, t % scn.W], kk[i, j, t].view(np.uint16))
                assert np.array_equal(p.win_v[u, t % scn.W], vv[i, j, t].view(np.uint16))
