"""NEXT-4: the three-level tier FP16-K8V4-K4V2 ("accommodating three precision levels can be achieved by
combining a unidirectional page table with a bidirectional one"; P:660 names FP16-K8V4-K4V2), readings Q38-Q44 of
DESIGN.md §3.  Pins of the oracle, all independent of its code:
  * reduction: a TOP threshold no significance reaches (alpha_t = 3e38) reproduces the two-level run byte for byte
    (decisions, ring, tables, counts, pages) and never touches the TOP table;
  * brute force: an independent list model of the three-level policy (sections as lists of (significance,
    position); Algorithm 1 one level up, Q39; one unidirectional + one bidirectional table, Q41; scan-ordered grants
    with a unit's TOP pages first, Q43) run side by side with the oracle over randomized tiny lifecycles with
    thresholds hit exactly, duplicates, frees and re-admissions: identical tables, ring, pointers, counts and
    per-slot (significance, position) after every call;
  * FP16 storage: every TOP slot holds the generator's fp16 K and V rows of its position bit for bit (Q40), and a
    TOP victim moved down holds exactly orc_quantize of those fp16 values (Q42);
  * invariants of PIN-10 extended to the TOP table, demand <= 1 page per unit per step, and the
    configurations the tier rejects (Q38, Q43, Q44)."""
import numpy as np
import pytest

import oracle
from tests import harness as H

IDLE, ADMITTING, ACTIVE, PENDING = 0, 1, 2, 3
TOP = 4


def f32(x):
    return np.float32(x)


def _scn(**kw):
    base = dict(R=3, Ly=2, H=2, d=32, M=160, W=8, Ch=4, Cl=8, P=4000, seed=7, top_tier=1, alpha_t=2.0, Ct=4)
    base.update(kw)
    return H.TINY.replace(**base)


def _lifecycle(scn, steps=30, frees=((12, [1]),), readmit=(16, 1, 50), lens=(70, 40, 100)):
    o = H.OracleBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    snaps = []
    H.admit([o], inp, life, list(range(len(lens))), list(lens))
    snaps.append(("prefill", o.snapshot(), None))
    frees = dict(frees)
    for step in range(steps):
        decs = H.decode_step([o], inp, life, step)
        snaps.append((f"step {step}", o.snapshot(), decs[0].copy()))
        if step in frees:
            H.free([o], life, frees[step])
        if readmit and step == readmit[0]:
            H.admit([o], inp, life, [readmit[1]], [readmit[2]])
            snaps.append(("readmit", o.snapshot(), None))
    return o, life, snaps


def test_unreachable_top_threshold_reproduces_two_levels():
    two = _scn(top_tier=0, alpha_t=0.0)
    three = _scn(alpha_t=3.0e38, Ct=2)                          # an FP16 page fits the unified page
    o2, _, s2 = _lifecycle(two)
    o3, _, s3 = _lifecycle(three)
    assert o2.page_bytes == o3.page_bytes
    for (w, a, da), (_, b, db) in zip(s2, s3):
        for k in ("ring", "start", "free", "table", "n_h", "n_l", "req_state", "seq_len", "win_k", "win_v", "pages"):
            assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (w, k)
        if da is not None:
            assert np.array_equal(da.view(np.uint8), db.view(np.uint8)), w
        assert (b["ttable"] == -1).all() and (b["n_t"] == 0).all(), w


def test_invariants_fp16_storage_and_demand():
    scn = _scn()
    o, life, snaps = _lifecycle(scn, steps=40)
    inp = H.Inputs(scn)
    p = o.pool
    seen_top = False
    for where, snap, dec in snaps:
        H.check_invariants(snap, scn, o.L, o.geom, life=None)
        if dec is not None:
            assert (dec["demand"] <= 1).all()
            assert set(np.unique(dec["grow"]).tolist()) <= {0, 1, 2, 3}
            seen_top |= bool((dec["tc_class"] == TOP).any())
    assert seen_top and (p.n_t > 0).any()
    # every TOP slot holds the fp16 K / V rows of its position exactly (Q40): prompt tokens from the prefill
    # generator, generated tokens from the decode generator (new token at position N - 1)
    g = p.geom[TOP]
    for u in range(p.U):
        r = u // p.LyH
        if p.req_state[r] != ACTIVE:
            continue
        for s in range(int(p.n_t[u])):
            pid, idx = p.slot_location(TOP, u, s)
            pg = p.pages[pid]
            pos = int(pg[g.off_pos + 4 * idx: g.off_pos + 4 * idx + 4].view(np.int32)[0])
            kr = pg[g.off_k + idx * g.k_row: g.off_k + (idx + 1) * g.k_row].view(np.uint16)
            vr = pg[g.off_v + idx * g.v_row: g.off_v + (idx + 1) * g.v_row].view(np.uint16)
            T0 = 50 if r == 1 else (70, 40, 100)[r]                   # prompt length (request 1 re-admitted)
            if pos < T0:
                _, k, v = inp.prefill([r], [T0])
                jk = k[0, u - r * p.LyH, pos].numpy().view(np.uint16)
                jv = v[0, u - r * p.LyH, pos].numpy().view(np.uint16)
            else:
                import synth
                ug = inp.ug.reshape(-1)[u:u + 1]
                import torch
                kk, vv = synth.new_token_kv(scn.seed, ug, torch.tensor([pos]), scn.d)
                jk, jv = kk[0].numpy().view(np.uint16), vv[0].numpy().view(np.uint16)
            assert np.array_equal(kr, jk) and np.array_equal(vr, jv), (u, s, pos)


def test_top_victim_moves_down_requantized_from_fp16():
    """Q42: a TOP victim leaving its section is quantized from its exact fp16 values at the destination class"""
    # prompt thresholds alpha / n (Q4's second reading) keep stored TOP significance near alpha_t / N, so the drift
    # of the stored scores pushes TOP minima below the decode threshold
    scn = _scn(alpha_t=1.5, alpha_h=1.0, alpha_l=0.3, seed=11, prompt_denominator=1)
    o = H.OracleBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o], inp, life, [0, 1, 2], [90, 90, 90])
    p = o.pool
    moved = 0
    for step in range(60):
        o.drift(step)                                             # the significance drift, then the step itself
        before = {(u, s): p.slot_record(TOP, u, s) for u in range(p.U) for s in range(int(p.n_t[u]))}
        fp16 = {}
        g = p.geom[TOP]
        for (u, s) in before:
            pid, idx = p.slot_location(TOP, u, s)
            pg = p.pages[pid]
            fp16[(u, s)] = (pg[g.off_k + idx * g.k_row: g.off_k + (idx + 1) * g.k_row].view(np.float16).astype(np.float32),
                            pg[g.off_v + idx * g.v_row: g.off_v + (idx + 1) * g.v_row].view(np.float16).astype(np.float32))
        decs = H.decode_step([o], inp, life, step, drift=False)
        dec = decs[0]
        for u in np.nonzero((dec["tc_class"] == TOP) & (dec["v_action"] == oracle.V_DOWN))[0]:
            u = int(u)
            dst = int(dec["grow"][u])
            kx, vx = fp16[(u, int(dec["v_slot"][u]))]
            kc, km, vc, vm, sg, ps = p.slot_record(dst, u, int(dec["v_dst_slot"][u]))
            gd = p.geom[dst]
            stk, ck, sk, zk = oracle.quantize(kx, gd.kbits)
            stv, cv, sv, zv = oracle.quantize(vx, gd.vbits)
            assert stk == 0 and stv == 0
            assert np.array_equal(kc, ck) and np.array_equal(vc, cv), (step, u)
            assert km == sk | (zk << 16) and vm == sv | (zv << 16), (step, u)
            assert (sg, ps) == before[(u, int(dec["v_slot"][u]))][4:], (step, u)
            moved += 1
    assert moved > 0


def test_rejected_configurations():
    for bad in (dict(alpha_t=0.5), dict(prefill_workflow=1), dict(Ct=0)):
        cfg = oracle.make_config(**_scn(**bad).config_dict())
        with pytest.raises(ValueError):
            oracle.OraclePool(cfg)
    o = H.OracleBackend(_scn(q_per_kv=2))
    q = np.zeros((o.U, 2, 32), np.float16)
    assert o.pool.attend(q)[0] == oracle.ERR_INVALID              # Q44: no NEXT-2 attention with the FP16 tier
    ah = np.full(o.pool.LyH, 3.0, np.float32)                     # per-head alpha_h above alpha_t (Q38)
    assert o.pool.set_head_thresholds(ah, np.zeros_like(ah)) == oracle.ERR_INVALID


# ------------------------------------------------------------------------------------------ brute force
class Model3:
    """Sections {TOP, 1 high, 2 low} as lists of (significance, position); the TOP table is unidirectional
    (left to right, Ct tokens per page), the bidirectional table as in the paper."""

    def __init__(self, R, LyH, W, Ct, Ch, Cl, P, M, at, ah, al):
        self.R, self.LyH, self.W, self.Ct, self.Ch, self.Cl, self.P, self.M = R, LyH, W, Ct, Ch, Cl, P, M
        self.at, self.ah, self.al = f32(at), f32(ah), f32(al)
        self.U = R * LyH
        self.L = -(-M // Ch) + (1 if W < Ch else 0)
        self.Lt = -(-M // Ct)
        self.ring = list(range(P))
        self.start, self.free = 0, P
        self.table = [[-1] * self.L for _ in range(self.U)]
        self.ttable = [[-1] * self.Lt for _ in range(self.U)]
        self.sec = [{TOP: [], 1: [], 2: []} for _ in range(self.U)]
        self.state = [IDLE] * R
        self.seq = [0] * R
        self.status = 0

    def C(self, cls):
        return {TOP: self.Ct, 1: self.Ch, 2: self.Cl}[cls]

    def cls_of(self, s, den):
        if s >= self.at / den:
            return TOP
        if s >= self.ah / den:
            return 1
        if s >= self.al / den:
            return 2
        return 3

    def _recycle(self):
        for r in range(self.R):
            if self.state[r] != PENDING:
                continue
            for u in range(r * self.LyH, (r + 1) * self.LyH):
                for row in (self.ttable[u], self.table[u]):             # Q41: TOP slots first
                    for k in range(len(row)):
                        if row[k] != -1:
                            self.ring[(self.start + self.free) % self.P] = row[k]
                            self.free += 1
                            row[k] = -1
                self.sec[u] = {TOP: [], 1: [], 2: []}
            self.state[r], self.seq[r] = IDLE, 0

    def _take(self, n):
        ids = [self.ring[(self.start + k) % self.P] for k in range(n)]
        self.start = (self.start + n) % self.P
        self.free -= n
        return ids

    def plan(self, lens, sig, reqs):
        plans = {}
        for i, r in enumerate(reqs):
            for j in range(self.LyH):
                secs = {TOP: [], 1: [], 2: []}
                for t in range(max(lens[i] - self.W, 0)):
                    s = f32(sig[i][j][t]) + f32(0)
                    c = self.cls_of(s, f32(t + 1))
                    if c != 3:
                        secs[c].append((s, t))
                plans[r * self.LyH + j] = secs
        return plans

    def prefill(self, reqs, lens, sig):
        plans = self.plan(lens, sig, reqs)
        for r in reqs:
            self.state[r] = ADMITTING
        self._recycle()
        D = sum(sum(-(-len(sc[c]) // self.C(c)) for c in sc) for sc in plans.values())
        if D > self.free:
            self.status = oracle.ERR_OOM
            return False
        for u in sorted(plans):
            sc = plans[u]
            pt, ph, pl = (-(-len(sc[c]) // self.C(c)) for c in (TOP, 1, 2))
            ids = self._take(pt + ph + pl)                              # Q43: TOP, high, low
            for k in range(pt):
                self.ttable[u][k] = ids[k]
            for k in range(ph):
                self.table[u][k] = ids[pt + k]
            for k in range(pl):
                self.table[u][self.L - 1 - k] = ids[pt + ph + k]
            self.sec[u] = {c: list(sc[c]) for c in sc}
        for i, r in enumerate(reqs):
            self.seq[r] = lens[i]
            self.state[r] = ACTIVE
        return True

    def decode(self, cand):
        self._recycle()
        grows = {}
        for u in range(self.U):
            r = u // self.LyH
            if self.state[r] != ACTIVE:
                continue
            N = self.seq[r] + 1
            pc = N - 1 - self.W
            if pc < 0:
                continue
            s = f32(cand[u]) + f32(0)
            cls = self.cls_of(s, f32(N))
            if cls == 3:
                continue
            bar = {TOP: self.at, 1: self.ah, 2: self.al}[cls] / f32(N)
            sec = self.sec[u][cls]
            v, p, k = min([(x, q, kk) for kk, (x, q) in enumerate(sec)] + [(s, pc, -1)], key=lambda x: (x[0], x[1]))
            if k == -1 or v >= bar:                                       # t_v stays: t_c appended
                grows[u] = (cls, "append", (s, pc))
            else:
                dest = self.cls_of(v, f32(N))                              # Q39: where t_v's score qualifies
                if dest == 3:
                    grows[u] = (None, "replace", (cls, k, (s, pc)))
                else:
                    grows[u] = (dest, "down", (cls, k, (s, pc), (v, p)))
        demand = {u: len(self.sec[u][g[0]]) % self.C(g[0]) == 0 for u, g in grows.items() if g[0] is not None}
        if sum(demand.values()) > self.free:
            self.status = oracle.ERR_OOM
            return
        for u in sorted(demand):
            if demand[u]:
                gcls = grows[u][0]
                n = len(self.sec[u][gcls])
                (pid,) = self._take(1)
                if gcls == TOP:
                    self.ttable[u][n // self.Ct] = pid
                else:
                    self.table[u][n // self.Ch if gcls == 1 else self.L - 1 - n // self.Cl] = pid
        for u, (gcls, kind, x) in grows.items():
            if kind == "append":
                self.sec[u][gcls].append(x)
            elif kind == "down":
                cls, k, tc, v = x
                self.sec[u][cls][k] = tc
                self.sec[u][gcls].append(v)
            else:
                cls, k, tc = x
                self.sec[u][cls][k] = tc
        for r in range(self.R):
            if self.state[r] == ACTIVE:
                self.seq[r] += 1


def _compare(m, pool, where):
    assert pool.status == m.status, where
    assert (pool.start, pool.free) == (m.start, m.free), where
    assert np.array_equal(pool.ring, np.array(m.ring, np.int32)), where
    assert np.array_equal(pool.table, np.array(m.table, np.int32).reshape(m.U, m.L)), where
    assert np.array_equal(pool.ttable, np.array(m.ttable, np.int32).reshape(m.U, m.Lt)), where
    for u in range(m.U):
        for cls, n in ((TOP, pool.n_t[u]), (1, pool.n_h[u]), (2, pool.n_l[u])):
            assert int(n) == len(m.sec[u][cls]), (where, u, cls)
            for s in range(int(n)):
                _, _, _, _, sg, ps = pool.slot_record(cls, u, s)
                v, p = m.sec[u][cls][s]
                assert (sg, ps) == (int(np.float32(v).view(np.uint32)), p), (where, u, cls, s)
    ids = [m.ring[(m.start + k) % m.P] for k in range(m.free)] + \
        [x for row in m.table + m.ttable for x in row if x >= 0]
    assert sorted(ids) == list(range(m.P)), where


def _lattice(rng, tt, th, tl, size):
    vals = np.array([0.0, tl, th, tt, 2 * tt, (tt + th) / 2, th / 2, tl / 2, (th + tl) / 2], np.float32)
    return vals[rng.integers(0, len(vals), size=size)]


@pytest.mark.parametrize("Ct,Ch,W", [(1, 1, 0), (2, 1, 1), (1, 2, 2), (4, 2, 1)])
def test_bruteforce_three_level_lifecycles(Ct, Ch, W):
    rng = np.random.default_rng(1000 + 100 * Ct + 10 * Ch + W)
    at, ah, al = 2.0, 1.0, 0.25
    for case in range(120):
        R, H_ = int(rng.choice([1, 2, 3])), int(rng.choice([1, 2]))
        if R * H_ > 3:
            H_ = 1
        P, M, Cl = int(rng.integers(5, 16)), 12, 2 * Ch
        cfg = oracle.make_config(R=R, Ly=1, H=H_, d=8, M=M, W=W, Ch=Ch, Cl=Cl, P=P, alpha_h=ah, alpha_l=al,
                                 top_tier=1, alpha_t=at, Ct=Ct)
        pool = oracle.OraclePool(cfg)
        m = Model3(R, H_, W, Ct, Ch, Cl, P, M, at, ah, al)
        U = R * H_
        zeros = lambda *shape: np.zeros(shape + (8,), np.float16)

        def admit(reqs):
            lens = [int(rng.integers(0, 7)) for _ in reqs]
            stride = max(max(lens), 1)
            sig = np.zeros((len(reqs), H_, stride), np.float32)
            for t in range(stride):
                d = f32(t + 1)
                sig[:, :, t] = _lattice(rng, f32(at) / d, f32(ah) / d, f32(al) / d, (len(reqs), H_))
            plans = m.plan(lens, sig, reqs)
            D = sum(sum(-(-len(sc[c]) // m.C(c)) for c in sc) for sc in plans.values())
            rec = sum(1 for r in range(R) if m.state[r] == PENDING
                      for u in range(r * H_, (r + 1) * H_) for row in (m.table[u], m.ttable[u]) for x in row if x >= 0)
            if D > m.free + rec:
                return False
            st, _ = pool.classify_prefill(reqs, lens, sig)
            assert st == 0 and pool.compact_alloc(None) == 0
            k = zeros(len(reqs), H_, stride)
            assert pool.quant_write_prefill(k, k, sig) == 0
            assert m.prefill(reqs, lens, sig)
            return True

        for r in range(R):
            admit([r])
        _compare(m, pool, f"case {case} admit")
        for step in range(8):
            if any(m.seq[r] >= M for r in range(R) if m.state[r] == ACTIVE):
                break
            cand = np.zeros(U, np.float32)
            for u in range(U):
                n = f32(m.seq[u // H_] + 1)
                cand[u] = _lattice(rng, f32(at) / n, f32(ah) / n, f32(al) / n, 1)[0]
            st, dec = pool.classify_decode(cand)
            assert st == 0 and pool.compact_alloc(dec) == 0
            k = np.zeros((U, 8), np.float16)
            assert pool.quant_write_decode(dec, k, k, cand) == 0
            m.decode(cand)
            _compare(m, pool, f"case {case} step {step}")
            if m.status:
                break
            act = [r for r in range(R) if m.state[r] == ACTIVE]
            if act and rng.random() < 0.3:
                fr = [int(x) for x in rng.choice(act, size=int(rng.integers(1, len(act) + 1)), replace=False)]
                assert pool.free_requests(fr) == 0
                for r in fr:
                    m.state[r] = PENDING
            idle = [r for r in range(R) if m.state[r] == IDLE]
            if idle and rng.random() < 0.3:
                admit([idle[0]])
                _compare(m, pool, f"case {case} re-admit {step}")
