"""Pins for the oracle's scalar arithmetic: IEEE binary16 conversion and the §2.2 quantizer.

The FP16 conversion is pinned against numpy.float16 (an independent implementation); the quantizer
against closed forms fixed by P:175-177 (Q = round((X - z)/s), X^ = s*Q + z, s and z from X_min and
X_max, kept in FP16) — see DESIGN.md §4 PIN-8.
"""
import numpy as np
import pytest

import oracle

pytestmark = []


def test_f32_from_f16_all_patterns():
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = h.view(np.float16).astype(np.float32)
    got = np.array([oracle.f32_from_f16(int(x)) for x in h[::7]], dtype=np.float32)
    r = ref[::7]
    nan = np.isnan(r)
    assert np.array_equal(got[~nan].view(np.uint32), r[~nan].view(np.uint32))
    assert np.isnan(got[nan]).all()


def test_f16_roundtrip_all_patterns():
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    f = h.view(np.float16).astype(np.float32)
    back = oracle.f16_from_f32_array(f)
    nan = np.isnan(f)
    assert np.array_equal(back[~nan], h[~nan])
    assert np.isnan(back[nan].view(np.float16)).all()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_f16_rne_random_fp32_bits(seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2 ** 32, size=1_000_000, dtype=np.uint64).astype(np.uint32)
    f = bits.view(np.float32)
    f = f[np.isfinite(f)]
    got = oracle.f16_from_f32_array(f)
    with np.errstate(over="ignore"):
        ref = f.astype(np.float16).view(np.uint16)
    assert np.array_equal(got, ref)


def test_f16_rne_near_halfway_and_boundaries():
    # values within a few ulps of every binary16 halfway point, plus the overflow / subnormal edges
    h = np.arange(0, 0x7C00, dtype=np.uint32).astype(np.uint16)
    lo = h.view(np.float16).astype(np.float64)
    hi = (h + 1).astype(np.uint16).view(np.float16).astype(np.float64)
    mid = ((lo + hi) / 2).astype(np.float32)
    cands = np.concatenate([mid, np.nextafter(mid, np.float32(0)), np.nextafter(mid, np.float32(np.inf)),
                            np.array([65504, 65519.99, 65520, 65536, 2.0 ** -24, 2.0 ** -25, 2.0 ** -25 * 1.0001,
                                      2.0 ** -14, 2.0 ** -14 - 2.0 ** -25], dtype=np.float32)])
    cands = np.concatenate([cands, -cands])
    got = oracle.f16_from_f32_array(cands)
    with np.errstate(over="ignore"):
        ref = cands.astype(np.float16).view(np.uint16)
    assert np.array_equal(got, ref)


def _q(x, bits):
    st, codes, s, z = oracle.quantize(np.asarray(x, np.float32), bits)
    assert st == oracle.OK
    return oracle.unpack_codes(codes, len(x), bits), s, z, codes


def test_quant_grid_example():
    # [0,1,2,3] at 2 bits -> s = 1, z = 0, codes [0,1,2,3]; dequantization exact (S:154 / P:175-176)
    q, s, z, codes = _q([0, 1, 2, 3], 2)
    assert list(q) == [0, 1, 2, 3]
    assert oracle.f32_from_f16(s) == 1.0 and oracle.f32_from_f16(z) == 0.0
    assert np.array_equal(oracle.dequantize(codes, 4, 2, s, z), np.array([0, 1, 2, 3], np.float32))
    # packing, Q17: lowest index in the least-significant bits: 0 | 1<<2 | 2<<4 | 3<<6
    assert codes[0] == 0b11100100


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quant_constant_vector_exact(bits):
    for c in (0.0, -0.0, 1.5, -3.25, 1e-5, 60000.0):
        x = np.full(16, np.float32(np.float16(c)), np.float32)
        q, s, z, codes = _q(x, bits)
        assert (q == 0).all() and oracle.f32_from_f16(s) == 0.0
        assert np.array_equal(oracle.dequantize(codes, 16, bits, s, z), x)


def _fp16_vectors(rng, n, d, scale=1.0):
    return (rng.standard_normal((n, d)) * scale).astype(np.float16).astype(np.float32)


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quant_error_bound_and_full_range(bits):
    rng = np.random.default_rng(bits)
    Q = (1 << bits) - 1
    for x in _fp16_vectors(rng, 3000, 64):
        q, s, z, codes = _q(x, bits)
        sf, zf = oracle.f32_from_f16(s), oracle.f32_from_f16(z)
        xh = oracle.dequantize(codes, 64, bits, s, z)
        if (x.max() - x.min()) / Q >= 2.0 ** -14:        # s32 in binary16's normal range
            assert np.abs(x - xh).max() <= sf / 2          # |x - x^| <= s/2
            assert q.min() == 0 and q.max() == Q           # non-constant input spans the code range
        assert zf == x.min()                               # z = X_min exactly for FP16 input
        assert (q >= 0).all() and (q <= Q).all()


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quant_error_bound_tiny_ranges(bits):
    rng = np.random.default_rng(100 + bits)
    Q = (1 << bits) - 1
    for _ in range(2000):
        base = np.float32(rng.standard_normal())
        span = 10.0 ** rng.uniform(-7, -1.5)
        x = (base + rng.uniform(0, span, 32)).astype(np.float16).astype(np.float32)
        q, s, z, codes = _q(x, bits)
        xh = oracle.dequantize(codes, 32, bits, s, z)
        assert np.abs(x - xh).max() <= oracle.f32_from_f16(s) / 2 + Q * 2.0 ** -25 + 1e-12


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quant_monotone_and_idempotent(bits):
    rng = np.random.default_rng(7 + bits)
    for x in _fp16_vectors(rng, 500, 128, 2.0):
        q, s, z, codes = _q(x, bits)
        order = np.argsort(x, kind="stable")
        assert (np.diff(q[order]) >= 0).all()              # monotone in x
        xh = oracle.dequantize(codes, 128, bits, s, z)
        q2, s2, z2, codes2 = _q(xh, bits)                  # quant -> dequant -> quant is a fixed point
        assert np.array_equal(q2, q) and s2 == s and z2 == z


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quant_power_of_two_invariance(bits):
    rng = np.random.default_rng(11 + bits)
    for x in _fp16_vectors(rng, 500, 64):
        q, _, _, _ = _q(x, bits)
        for k in (-3, 2):
            q2, _, _, _ = _q((x * np.float32(2.0 ** k)).astype(np.float32), bits)
            assert np.array_equal(q, q2)


def test_quant_rounding_half_away_from_zero():
    # x = [0, 0.5, 1, 1.5, 2, 2.5, 3, 3] at 2 bits: s = 1, z = 0; 0.5 -> 1, 1.5 -> 2, 2.5 -> 3
    q, s, z, _ = _q([0, 0.5, 1, 1.5, 2, 2.5, 3, 3], 2)
    assert list(q) == [0, 1, 1, 2, 2, 3, 3, 3]


def test_quant_nonfinite_rejected():
    for bad in (np.inf, -np.inf, np.nan):
        st, *_ = oracle.quantize(np.array([0, 1, bad, 2], np.float32), 4)
        assert st == oracle.ERR_NONFINITE


def test_downgrade_is_quantize_of_dequantized():
    # Q9 / S:169: the K4V2 copy of a K8V4 token is quant(dequant(codes8), 4 bits)
    rng = np.random.default_rng(5)
    for x in _fp16_vectors(rng, 200, 64):
        _, s8, z8, c8 = _q(x, 8)
        xh = oracle.dequantize(c8, 64, 8, s8, z8)
        q4, s4, z4, _ = _q(xh, 4)
        assert q4.max() <= 15
        # the 4-bit reconstruction stays within s4/2 (+ fp16 rounding of z) of the 8-bit one
        _, _, _, c4 = _q(xh, 4)
        x4 = oracle.dequantize(c4, 64, 4, s4, z4)
        assert np.abs(x4 - xh).max() <= oracle.f32_from_f16(s4) / 2 + abs(oracle.f32_from_f16(z4)) * 2 ** -10 + 1e-6
