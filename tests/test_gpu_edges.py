"""GPU-vs-oracle parity on the degenerate and failure cases of the path (DESIGN.md §1 error model):
all-or-nothing OOM in decode and prefill (Q15) with recovery by freeing and re-issuing dkv_compact_alloc,
non-finite significance / K / V (sticky DKV_ERR_NONFINITE, later calls no-ops), steps with no active
request, empty admissions, prompts no longer than the window (Q22), requests run up to max_seq_len, and
alpha = 0 / all-pruned thresholds (PIN-6 / PIN-7 at GPU level)."""
import numpy as np
import pytest
import torch

import oracle
from tests import harness as H

pytestmark = pytest.mark.gpu


def _pair(scn):
    from tests.gpu_backend import GpuBackend
    return H.OracleBackend(scn), GpuBackend(scn)


def _signed(x):
    return x - (1 << 32) if x >= (1 << 31) else x


def _same(o, g, where, pages=True):
    from tests.gpu_backend import compare_state
    so, sg = o.snapshot(pages=pages), g.snapshot(pages=pages)
    compare_state(so, sg, where=where)
    assert o.pool.status == _signed(sg["status"]), (where, o.pool.status, sg["status"])


def _step(o, g, inp, life, step, check=True):
    """one decode step on both backends; returns the decisions (oracle, gpu)"""
    from tests.gpu_backend import dec_np
    decs = H.decode_step([o, g], inp, life, step)
    if check:
        a, b = dec_np(decs[0]), dec_np(decs[1])
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"decisions differ at step {step}"
        _same(o, g, f"step {step}")
    return decs


def _used_after_prefill(scn, lens):
    o = H.OracleBackend(scn.replace(P=1 << 16))
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o], inp, life, list(range(len(lens))), lens)
    return (1 << 16) - o.pool.free, o, inp, life


def _pool_pages_for_second_oom(scn, lens):
    """pages for which an admission of `lens` succeeds and a second, identical one runs out: the first needs
    its transient demand (the prompt workflow's conservative blocks exceed what it keeps, Fig. 5)"""
    used, o, _, _ = _used_after_prefill(scn, lens)
    return max(used + 5, int(o.pool.last_demand) + 2)


def test_decode_oom_all_or_nothing_then_recover():
    from tests.gpu_backend import dec_np
    scn = H.TINY
    used, _, _, _ = _used_after_prefill(scn, [64] * 4)
    scn = scn.replace(P=used + 3)                  # a few decode pages, then OOM
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [0, 1, 2, 3], [64] * 4)
    _same(o, g, "prefill")
    for step in range(64):
        active = life.state == H.REQ_ACTIVE
        N = np.where(active, life.seq + 1, 0)
        for b in (o, g):
            b.drift(step)
        cand, k, v = inp.decode(N)
        (_, do), (_, dg) = o.classify_decode(cand), g.classify_decode(cand)
        assert np.array_equal(dec_np(do).view(np.uint8), dec_np(dg).view(np.uint8))
        assert o.compact_alloc(do) == 0 and g.compact_alloc(dg) == 0
        if o.pool.status == oracle.ERR_OOM:
            _same(o, g, f"OOM at step {step}")       # allocation state unchanged on both sides
            assert o.take_status() == oracle.ERR_OOM and g.take_status() == oracle.ERR_OOM
            # recovery (dkv.h): free a request, re-issue compact_alloc with the same decisions
            assert o.free([2]) == 0 and g.free([2]) == 0
            assert o.compact_alloc(do) == 0 and g.compact_alloc(dg) == 0
            assert o.pool.status == 0
            assert o.quant_write_decode(do, k, v, cand) == 0 and g.quant_write_decode(dg, k, v, cand) == 0
            _same(o, g, f"recovered at step {step}")
            return
        assert o.quant_write_decode(do, k, v, cand) == 0 and g.quant_write_decode(dg, k, v, cand) == 0
        life.seq[active] += 1
        _same(o, g, f"step {step}", pages=step % 8 == 0)
    pytest.fail("the pool never ran out of pages")


@pytest.mark.parametrize("workflow", [0, 1])
def test_prefill_oom_leaves_allocation_untouched(workflow):
    scn = H.TINY.replace(prefill_workflow=workflow)
    scn = scn.replace(P=_pool_pages_for_second_oom(scn, [64, 64]))
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [0, 1], [64, 64])
    _same(o, g, "first admission")
    assert o.pool.status == 0
    sig, k, v = inp.prefill([2, 3], [64, 64])
    for b in (o, g):
        assert b.classify_prefill([2, 3], [64, 64], sig) == 0
        assert b.compact_alloc(None) == 0
    assert o.pool.status == oracle.ERR_OOM
    _same(o, g, "prefill OOM")
    for b in (o, g):
        assert b.quant_write_prefill(k, v, sig) == 0         # no-op under the sticky status
    _same(o, g, "quant_write after OOM")


@pytest.mark.parametrize("where", ["prefill_sig", "prefill_kv", "decode_sig", "decode_kv"])
def test_nonfinite_inputs_set_sticky_status(where):
    scn = H.TINY
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    if where.startswith("prefill"):
        sig, k, v = inp.prefill([0, 1], [64, 64])
        if where == "prefill_sig":
            sig = sig.clone()
            sig[1, 3, 7] = float("nan")
        else:                                              # Q30: the token is rejected whole, others written
            k = k.clone()
            k.view(torch.int16)[0, 5, 2, 11] = 0x7E00      # NaN in one element of a kept token's key
            k.view(torch.int16)[1, 0, 60, 0] = -1024       # 0xFC00 = -inf in a window token (copied, not quantized)
        for b in (o, g):
            assert b.classify_prefill([0, 1], [64, 64], sig) == 0
            assert b.compact_alloc(None) == 0
            assert b.quant_write_prefill(k, v, sig) == 0
        assert o.pool.status == oracle.ERR_NONFINITE
        _same(o, g, where)
        return
    H.admit([o, g], inp, life, [0, 1, 2, 3], [64] * 4)
    N = life.seq + 1
    cand, k, v = inp.decode(N)
    if where == "decode_sig":
        cand = cand.clone()
        cand[5] = -1.0
    else:
        v = v.clone()
        v.view(torch.int16)[9, 3] = 0x7C00             # +inf in the new token: it reaches t_c W steps later
    from tests.gpu_backend import dec_np
    for step in range(scn.W + 2):
        for b in (o, g):
            b.drift(step)
        (_, do), (_, dg) = o.classify_decode(cand), g.classify_decode(cand)
        for b, d in ((o, do), (g, dg)):
            assert b.compact_alloc(d) == 0
            assert b.quant_write_decode(d, k, v, cand) == 0
        _same(o, g, f"{where} step {step}", pages=True)
        if o.pool.status != 0:
            assert o.pool.status == oracle.ERR_NONFINITE
            return
        life.seq += 1
        cand, k2, v2 = inp.decode(life.seq + 1)
        k, v = k2, v2 if where != "decode_kv" else v2
    pytest.fail("non-finite input never detected")


def test_no_active_requests_and_empty_admission():
    scn = H.TINY
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [], [])                       # n = 0
    _same(o, g, "empty admission")
    for step in range(3):
        H.decode_step([o, g], inp, life, step)               # nothing active: every decision empty
        _same(o, g, f"idle step {step}")
    H.admit([o, g], inp, life, [0, 2], [16, 9])              # prompts <= W: nothing stored (Q22)
    _same(o, g, "window-only prompts")
    for step in range(20):                                    # t_c appears once N - 1 - W >= 0
        _step(o, g, inp, life, 100 + step)


def test_run_to_max_seq_len():
    scn = H.TINY.replace(M=96)
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [0, 1, 2, 3], [90, 64, 80, 95])
    for step in range(1):
        _step(o, g, inp, life, step)                          # request 3 reaches M = 96
    from paper_2412_03131_b200 import dkv as D
    cand, k, v = inp.decode(np.where(life.state == H.REQ_ACTIVE, life.seq + 1, 0))
    with pytest.raises(RuntimeError):
        g.classify_decode(cand)                               # DKV_ERR_STATE: an ACTIVE request is at M
    assert o.free([3]) == 0 and g.free([3]) == 0
    life.state[3] = H.REQ_PENDING_FREE
    for step in range(5):
        _step(o, g, inp, life, 10 + step)


@pytest.mark.parametrize("alphas", [(0.0, 0.0), (1.0e30, 1.0e30)])
def test_alpha_special_cases(alphas):
    # PIN-6 (alpha = 0: every candidate High, no victim ever leaves -> PagedAttention-style allocation) and
    # PIN-7 (alpha_l huge: everything pruned, no page ever allocated), GPU against the oracle
    scn = H.TINY.replace(alpha_h=alphas[0], alpha_l=alphas[1], R=3, Ly=2, H=6, M=256, P=3000, seed=9)
    o, g = _pair(scn)
    # significance drawn for the default thresholds (the generator follows the thresholds it is given)
    inp, life = H.Inputs(scn.replace(alpha_h=1.0, alpha_l=0.02)), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [0, 1, 2], [100, 64, 33])
    _same(o, g, "prefill")
    for step in range(40):
        _step(o, g, inp, life, step)
    if alphas[1] > 1e20:
        assert o.pool.free == scn.P


@pytest.mark.parametrize("workflow", [0, 1])
def test_prefill_error_rolls_back_admission_then_readmit(workflow):
    """a dkv_quant_write(PREFILL) that finds an error at entry (here the admission's OOM)
    rolls the admission back (ADMITTING -> IDLE, no pages held), so after dkv_pool_query the slots are
    re-admissible; GPU and oracle agree at every step."""
    scn = H.TINY.replace(prefill_workflow=workflow)
    scn = scn.replace(P=_pool_pages_for_second_oom(scn, [64, 64]))
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, [0, 1], [64, 64])
    assert o.pool.status == 0
    sig, k, v = inp.prefill([2, 3], [64, 64])
    for b in (o, g):
        assert b.classify_prefill([2, 3], [64, 64], sig) == 0
        assert b.compact_alloc(None) == 0
        assert b.quant_write_prefill(k, v, sig) == 0
    _same(o, g, "rolled back")
    assert list(o.pool.req_state[2:4]) == [H.REQ_IDLE, H.REQ_IDLE]
    assert o.take_status() == oracle.ERR_OOM and g.take_status() == oracle.ERR_OOM
    H.free([o, g], life, [0])                                  # make room, then admit a short prompt
    for step in range(2):
        _step(o, g, inp, life, step)
    H.admit([o, g], inp, life, [2], [40])
    _same(o, g, "re-admitted")
    for step in range(2, 6):
        _step(o, g, inp, life, step)


def test_prefill_nonfinite_token_request_active_and_freeable():
    """Q30/Q37: a non-finite K element found by the bulk writer rejects that token only; the requests become
    ACTIVE (sticky NONFINITE), so after the query they can be freed and their pages recycled."""
    scn = H.TINY
    o, g = _pair(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    sig, k, v = inp.prefill([0, 1], [64, 64])
    k = k.clone()
    k.view(torch.int16)[1, 2, 3, 5] = 0x7E00
    for b in (o, g):
        assert b.classify_prefill([0, 1], [64, 64], sig) == 0
        assert b.compact_alloc(None) == 0
        assert b.quant_write_prefill(k, v, sig) == 0
    _same(o, g, "prefill with a NaN key")
    assert list(o.pool.req_state[:2]) == [H.REQ_ACTIVE, H.REQ_ACTIVE]
    assert o.take_status() == oracle.ERR_NONFINITE and g.take_status() == oracle.ERR_NONFINITE
    for b in (o, g):
        assert b.free([0, 1]) == 0
    life.state[:] = H.REQ_IDLE
    H.decode_step([o, g], inp, life, 0)                          # recycles both requests
    _same(o, g, "freed")
    assert o.pool.free == scn.P
    H.admit([o, g], inp, life, [0, 1], [64, 50])
    _same(o, g, "re-admitted")


def test_nonfinite_multi_cta_units_keep_going():
    """the status is one snapshot per call, so an error found in one unit (one CTA) does not
    stop the units of CTAs that start later: a pool spanning many CTAs of every decode / prefill kernel, with
    non-finite significance and K/V in units far apart, matches the oracle in every byte."""
    scn = H.TINY.replace(R=16, Ly=4, H=8, d=64, M=256, W=16, P=40000, seed=17)
    for where in ("decode_kv", "decode_sig", "prefill_kv"):
        o, g = _pair(scn)
        inp, life = H.Inputs(scn), H.Lifecycle(scn)
        reqs = list(range(scn.R))
        lens = [80 + 7 * r for r in reqs]
        if where == "prefill_kv":
            sig, k, v = inp.prefill(reqs, lens)
            k = k.clone()
            for (i, j, t) in ((0, 1, 3), (7, 30, 40), (15, 31, 60)):
                k.view(torch.int16)[i, j, t, 9] = 0x7C00
            for b in (o, g):
                assert b.classify_prefill(reqs, lens, sig) == 0
                assert b.compact_alloc(None) == 0
                assert b.quant_write_prefill(k, v, sig) == 0
            _same(o, g, where)
            assert o.pool.status == oracle.ERR_NONFINITE
            continue
        H.admit([o, g], inp, life, reqs, lens)
        N = life.seq + 1
        cand, k, v = inp.decode(N)
        bad = [3, scn.U // 2 + 5, scn.U - 2]
        if where == "decode_sig":
            cand = cand.clone()
            cand[bad] = float("nan")
        else:
            k = k.clone()
            for u in bad:
                k.view(torch.int16)[u, 7] = 0x7E00              # reaches t_c W steps later
        from tests.gpu_backend import dec_np
        for step in range(scn.W + 2):
            (_, do), (_, dg) = o.classify_decode(cand), g.classify_decode(cand)
            assert np.array_equal(dec_np(do).view(np.uint8), dec_np(dg).view(np.uint8)), (where, step)
            for b, d in ((o, do), (g, dg)):
                assert b.compact_alloc(d) == 0
                assert b.quant_write_decode(d, k, v, cand) == 0
            _same(o, g, f"{where} step {step}", pages=True)
            if o.pool.status != 0:
                break
            life.seq += 1
            cand, k2, v2 = inp.decode(life.seq + 1)
            k = k2 if where != "decode_kv" else k
            v = v2
        assert o.pool.status == oracle.ERR_NONFINITE, where
