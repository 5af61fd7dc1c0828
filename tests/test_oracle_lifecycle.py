"""Oracle lifecycle pins: invariants after every call (PIN-10), Algorithm 1 restated literally with sets
(PIN-4), per-step demand (PIN-5), the PagedAttention reduction (PIN-6), all-pruned (PIN-7), the allocation
order = exclusive scan over canonical units (PIN-9) and all-or-nothing OOM (Q15)."""
import itertools

import numpy as np
import pytest

import oracle
from tests import harness as H

TINY = H.TINY


def _run(scn, steps=64, frees=(), readmit_after=2, prompt=64, check_every=True, on_step=None, gen_scn=None):
    o = H.OracleBackend(scn)
    inp = H.Inputs(gen_scn or scn)
    life = H.Lifecycle(scn)
    reqs = list(range(scn.R))
    H.admit([o], inp, life, reqs, [prompt] * len(reqs))
    H.check_invariants(o.snapshot(), scn, o.L, o.geom, life)
    pending = {}
    for step in range(steps):
        snap_before = o.snapshot(pages=False)
        decs = H.decode_step([o], inp, life, step)
        if on_step:
            on_step(step, o, snap_before, decs[0], life)
        if check_every:
            H.check_invariants(o.snapshot(), scn, o.L, o.geom, life)
        for r, t in list(pending.items()):
            if step >= t and o.pool.req_state[r] == oracle.REQ_IDLE:
                H.admit([o], inp, life, [r], [prompt // 2 + 3])
                del pending[r]
        if step in dict(frees):
            rs = dict(frees)[step]
            H.free([o], life, rs)
            for r in rs:
                pending[r] = step + readmit_after
    return o, life


def test_tiny_lifecycle_invariants():
    _run(TINY, steps=64, frees=[(32, [1])])


@pytest.mark.parametrize("seed", [2, 3, 4, 5])
def test_random_lifecycles_invariants(seed):
    scn = TINY.replace(seed=seed, R=3, Ly=2, H=3, d=32, W=4, Ch=4, Cl=8, M=96, P=400,
                       alpha_h=1.0 + seed % 2, alpha_l=0.02 * (seed % 3))
    _run(scn, steps=60, frees=[(10, [0]), (25, [2]), (40, [1])], prompt=24)


def test_demand_at_most_one_page_and_predicted():
    # "a head allocates a new page only if either its high-precision or low-precision pages are
    # full, requiring at most one additional page per step"
    def on_step(step, o, before, dec, life):
        assert (dec["demand"] <= 1).all()
        grow_h = dec["grow"] == oracle.GROW_HIGH
        grow_l = dec["grow"] == oracle.GROW_LOW
        pred = (grow_h & (before["n_h"] % TINY.Ch == 0)) | (grow_l & (before["n_l"] % TINY.Cl == 0))
        assert np.array_equal(dec["demand"].astype(bool), pred)
        # "page recycling is not performed during generation" -> stored count grows by <= 1
        assert ((o.pool.n_h + o.pool.n_l) - (before["n_h"] + before["n_l"]) <= 1).all()
    _run(TINY, steps=64, on_step=on_step)


def test_allocation_order_is_exclusive_scan_of_demand():
    # each head reads its page IDs at a unique offset from the start pointer; offsets are the
    # exclusive prefix sum of per-head demand in canonical unit order (Q13) — itertools.accumulate here.
    def on_step(step, o, before, dec, life):
        dem = dec["demand"].astype(np.int64)
        off = [0] + list(itertools.accumulate(dem))[:-1]
        P = TINY.P
        for u in np.nonzero(dem)[0]:
            pid = before["ring"][(before["start"] + off[u]) % P]
            newrow = o.pool.table[u]
            oldrow = before["table"][u]
            changed = np.nonzero(newrow != oldrow)[0]
            assert len(changed) == 1 and newrow[changed[0]] == pid
        assert o.pool.start == (before["start"] + dem.sum()) % P
    _run(TINY, steps=64, on_step=on_step)


def test_paged_attention_reduction_alpha_zero():
    # PIN-6: alpha_h = alpha_l = 0 -> every candidate is High and no victim ever leaves; the pool then
    # behaves like PagedAttention block allocation: ph = ceil((N - W)/C_h), a new page every
    # C_h tokens, handed out in ring order across units in canonical order.
    scn = TINY.replace(alpha_h=0.0, alpha_l=0.0, R=1, P=1024, M=256)
    o = H.OracleBackend(scn)
    inp = H.Inputs(scn)
    life = H.Lifecycle(scn)
    H.admit([o], inp, life, [0], [scn.W])           # prompt entirely in the window: no pages yet
    assert o.pool.free == scn.P
    U = scn.U
    for step in range(96):
        H.decode_step([o], inp, life, step)
        N = life.seq[0]
        stored = max(N - scn.W, 0)
        assert (o.pool.n_h == stored).all() and (o.pool.n_l == 0).all()
        ph = -(-stored // scn.Ch)
        assert o.pool.free == scn.P - ph * U
        # page k of unit u is ring position k*U + u of the initial iota ring
        for k in range(ph):
            assert np.array_equal(o.pool.table[:, k], k * U + np.arange(U))


def test_all_pruned_allocates_nothing():
    # PIN-7: alpha_l huge -> every candidate below alpha_l/N -> pruned, free stays P forever
    scn = TINY.replace(alpha_h=1e30, alpha_l=1e30)
    o, life = _run(scn, steps=40, gen_scn=TINY)          # inputs drawn for the usual thresholds
    assert o.pool.free == scn.P and (o.pool.table == -1).all()


def test_all_or_nothing_oom():
    scn = TINY.replace(P=60)
    o = H.OracleBackend(scn)
    inp = H.Inputs(scn)
    life = H.Lifecycle(scn)
    H.admit([o], inp, life, [0, 1], [64, 64])
    # second admission does not fit: nothing may change except the status
    before = o.snapshot()
    sig, k, v = inp.prefill([2, 3], [64, 64])
    assert o.classify_prefill([2, 3], [64, 64], sig) == 0
    assert o.compact_alloc(None) == 0
    assert o.pool.status == oracle.ERR_OOM
    after = o.snapshot()
    for key in ("ring", "start", "free", "table", "n_h", "n_l"):
        assert np.array_equal(before[key], after[key]), key
    assert o.quant_write_prefill(k, v, sig) == 0       # no-op while the sticky status is set
    assert np.array_equal(before["pages"], o.snapshot()["pages"])
    assert o.take_status() == oracle.ERR_OOM and o.pool.status == 0


class LiteralAlgorithm1:
    """Algorithm 1 written with sets exactly as printed: KV_h.add(t_c); t_v = argmin; ...
    plus §4's prompt rule.  Tracks {position: significance} per unit; knows nothing about pages."""

    def __init__(self, scn):
        self.scn = scn
        self.kv_h = [dict() for _ in range(scn.U)]
        self.kv_l = [dict() for _ in range(scn.U)]

    def prompt(self, u, sig_row, n):
        s = self.scn
        for t in range(max(n - s.W, 0)):
            den = np.float32(t + 1) if s.prompt_denominator == 0 else np.float32(n)
            th, tl = np.float32(s.alpha_h) / den, np.float32(s.alpha_l) / den
            x = np.float32(sig_row[t]) + np.float32(0)      # -0 -> +0
            if x >= th:
                self.kv_h[u][t] = x
            elif x >= tl:
                self.kv_l[u][t] = x

    def step(self, u, N, sc):
        s = self.scn
        pc = N - 1 - s.W
        if pc < 0:
            return
        th, tl = np.float32(s.alpha_h) / np.float32(N), np.float32(s.alpha_l) / np.float32(N)
        sc = np.float32(sc) + np.float32(0)
        argmin = lambda sec: min(sec.items(), key=lambda kv: (kv[1], kv[0]))   # ties -> oldest (Q6)
        if sc >= th:
            self.kv_h[u][pc] = sc
            pv, sv = argmin(self.kv_h[u])
            if tl <= sv < th:
                del self.kv_h[u][pv]
                self.kv_l[u][pv] = sv
            elif sv < tl:
                del self.kv_h[u][pv]
        elif sc >= tl:
            self.kv_l[u][pc] = sc
            pv, sv = argmin(self.kv_l[u])
            if sv < tl:
                del self.kv_l[u][pv]

    def drift(self, step, ug):
        import torch
        import synth
        for u in range(self.scn.U):
            for sec in (self.kv_h[u], self.kv_l[u]):
                if not sec:
                    continue
                pos = np.array(sorted(sec), np.int64)
                f = synth.drift_factor(self.scn.seed, step, torch.full((len(pos),), int(ug[u])),
                                       torch.from_numpy(pos)).numpy()
                for p_, f_ in zip(pos, f):
                    sec[int(p_)] = np.float32(sec[int(p_)] * f_)


def _sections(o, u):
    p = o.pool
    out = []
    for cls, n in ((1, p.n_h[u]), (2, p.n_l[u])):
        d = {}
        for s in range(int(n)):
            _, _, _, _, sg, ps = p.slot_record(cls, u, s)
            d[ps] = np.uint32(sg).view(np.float32)
        out.append(d)
    return out


@pytest.mark.parametrize("seed,alpha", [(1, (1.0, 0.02)), (7, (3.0, 0.0)), (9, (1.0, 0.04))])
def test_oracle_matches_literal_algorithm1(seed, alpha):
    scn = TINY.replace(seed=seed, alpha_h=alpha[0], alpha_l=alpha[1], R=2, Ly=2, H=2, W=8, Ch=4, Cl=8, M=160, P=512)
    o = H.OracleBackend(scn)
    inp = H.Inputs(scn)
    life = H.Lifecycle(scn)
    lit = LiteralAlgorithm1(scn)
    sig = H.admit([o], inp, life, [0, 1], [40, 40])
    sg = H._np(sig)
    for r in range(2):
        for j in range(scn.LyH):
            lit.prompt(r * scn.LyH + j, sg[r, j], 40)
    ug = inp.ug.reshape(-1).numpy()

    def compare():
        for u in range(scn.U):
            h, l = _sections(o, u)
            assert h == lit.kv_h[u] and l == lit.kv_l[u], f"unit {u} differs from literal Algorithm 1"

    compare()
    for step in range(100):
        lit.drift(step, ug)
        N = life.seq + 1
        cand, _, _ = inp.decode(N)
        H.decode_step([o], inp, life, step)
        for u in range(scn.U):
            lit.step(u, int(N[u // scn.LyH]), float(cand[u]))
        compare()


def test_classify_prefill_matches_thresholds_bruteforce():
    # §4, P:363-366 with Q2 (half-open) on a lattice that hits the thresholds exactly
    for den_mode in (0, 1):
        scn = TINY.replace(R=1, Ly=1, H=1, W=2, prompt_denominator=den_mode, alpha_h=2.0, alpha_l=0.5)
        o = H.OracleBackend(scn)
        n = 12
        vals = np.float32([0.0, -0.0, 0.25, 0.5, 1.0, 2.0 / 3, 0.125, 2.0, 0.04166667, 0.5 / 11, 4.0, 0.1])
        sig = vals.reshape(1, 1, n)
        st, cls = o.pool.classify_prefill([0], [n], sig)
        assert st == 0
        for t in range(n):
            if t >= n - scn.W:
                assert cls[0, 0, t] == oracle.CLS_NONE
                continue
            den = np.float32(t + 1) if den_mode == 0 else np.float32(n)
            th, tl = np.float32(2.0) / den, np.float32(0.5) / den
            x = vals[t]
            want = oracle.CLS_HIGH if x >= th else oracle.CLS_LOW if x >= tl else oracle.CLS_PRUNED
            assert cls[0, 0, t] == want


def test_host_state_machine_errors():
    o = H.OracleBackend(TINY)
    inp = H.Inputs(TINY)
    life = H.Lifecycle(TINY)
    assert o.free([0]) == oracle.ERR_STATE                           # not active
    H.admit([o], inp, life, [0], [64])
    sig, _, _ = inp.prefill([0], [64])
    assert o.classify_prefill([0], [64], sig) == oracle.ERR_STATE    # already admitted
    assert o.free([0, 0]) == oracle.ERR_STATE                        # duplicate
    assert o.free([0]) == 0
    assert o.free([0]) == oracle.ERR_STATE                           # double free


def test_decode_page_contents():
    """quant_write(DECODE) pin: t_c's slot holds quantize(K/V of position p_c) at its class bits with
    score s_c and position p_c; a downgraded victim's KV_l slot holds quantize(dequantize(old KV_h
    record)) at the low bits with its score and position carried over (Q9)."""
    scn = TINY.replace(R=2)
    prompt = 40
    inp = H.Inputs(scn)
    _, kp, vp = inp.prefill([0, 1], [prompt, prompt])
    kp, vp = H._np(kp), H._np(vp)

    def kv_at(u, pos):
        r, j = divmod(u, scn.LyH)
        if pos < prompt:
            return kp[r, j, pos], vp[r, j, pos]
        import torch
        import synth
        k, v = synth.new_token_kv(scn.seed, inp.ug.reshape(-1)[u:u + 1], torch.tensor([pos]), scn.d)
        return H._np(k)[0], H._np(v)[0]

    def rec_q(cls, x, bits_key):
        g = oracle.OraclePool  # noqa
        return oracle.quantize(x.view(np.float16).astype(np.float32), bits_key)

    seen = {"down": 0, "tc": 0}

    def on_step(step, o, before, dec, life):
        p = o.pool
        cand, _, _ = inp.decode(np.where(life.state == 2, life.seq, 0))   # seq already advanced
        for u in range(scn.U):
            D = dec[u]
            N = int(life.seq[u // scn.LyH])
            pc = N - 1 - scn.W
            if D["tc_class"] in (1, 2):
                cls = int(D["tc_class"])
                kc, km, vc, vm, sg, ps = p.slot_record(cls, u, int(D["tc_slot"]))
                kx, vx = kv_at(u, pc)
                gm = p.geom[cls]
                _, ck, sk, zk = oracle.quantize(kx.view(np.float16).astype(np.float32), gm.kbits)
                _, cv, sv, zv = oracle.quantize(vx.view(np.float16).astype(np.float32), gm.vbits)
                assert np.array_equal(kc, ck) and np.array_equal(vc, cv) and ps == pc
                assert km == sk | (zk << 16) and vm == sv | (zv << 16)
                assert sg == int((np.float32(cand[u].item()) + np.float32(0)).view(np.uint32))
                seen["tc"] += 1
            if D["v_action"] == 2:
                # old high record from the snapshot taken before the step
                gh, gl = p.geom[1], p.geom[2]
                pid = before["table"][u, int(D["v_slot"]) // gh.C]
                idx = int(D["v_slot"]) % gh.C
                pg = before["pages"][pid]
                ks, kz = (int(pg[gh.off_kmeta + 4 * idx: gh.off_kmeta + 4 * idx + 4].view("<u2")[i]) for i in (0, 1))
                vs, vz = (int(pg[gh.off_vmeta + 4 * idx: gh.off_vmeta + 4 * idx + 4].view("<u2")[i]) for i in (0, 1))
                xk = oracle.dequantize(pg[gh.off_k + idx * gh.k_row:][:gh.k_row], scn.d, gh.kbits, ks, kz)
                xv = oracle.dequantize(pg[gh.off_v + idx * gh.v_row:][:gh.v_row], scn.d, gh.vbits, vs, vz)
                osg = int(pg[gh.off_score + 4 * idx: gh.off_score + 4 * idx + 4].view("<u4")[0])
                ops = int(pg[gh.off_pos + 4 * idx: gh.off_pos + 4 * idx + 4].view("<i4")[0])
                kc, km, vc, vm, sg, ps = p.slot_record(2, u, int(D["v_dst_slot"]))
                _, ck, sk, zk = oracle.quantize(xk, gl.kbits)
                _, cv, sv, zv = oracle.quantize(xv, gl.vbits)
                assert np.array_equal(kc, ck) and np.array_equal(vc, cv)
                assert km == sk | (zk << 16) and vm == sv | (zv << 16) and sg == osg and ps == ops
                seen["down"] += 1

    o = H.OracleBackend(scn)
    life = H.Lifecycle(scn)
    H.admit([o], inp, life, [0, 1], [prompt, prompt])
    for step in range(48):
        o.drift(step)
        before = o.snapshot()
        decs = H.decode_step([o], inp, life, step, drift=False)
        on_step(step, o, before, decs[0], life)
    assert seen["down"] > 0 and seen["tc"] > 0
