"""PIN-11: brute force on tiny pools.  An independent, list-based model of the method's metadata — sections as
lists of (significance, position) in slot order, the circular free list, the bidirectional tables — written
from the paper's statements (P:363-366 prompt classes, Algorithm 1 P:387-413 with readings Q2/Q3/Q6-Q8,
demand P:533-535, scan-ordered grants P:485-487 with Q13-Q15, recycling P:537) is run side by side with the
oracle over 1000 randomized tiny lifecycles (P <= 12 pages, 2-3 units, C_h in {1, 2, 4}, W in
{0, 1, 2}, significance from a lattice containing both thresholds exactly and many duplicates, random frees
and re-admissions, OOM).  After every call: identical tables, ring, pointers, counts and per-slot
(significance, position); every invariant of PIN-10 holds."""
import numpy as np
import pytest

import oracle

IDLE, ADMITTING, ACTIVE, PENDING = 0, 1, 2, 3


def f32(x):
    return np.float32(x)


class Model:
    def __init__(self, R, Ly, H, W, Ch, Cl, P, M, ah, al):
        self.R, self.LyH, self.W, self.Ch, self.Cl, self.P, self.M = R, Ly * H, W, Ch, Cl, P, M
        self.ah, self.al = f32(ah), f32(al)
        self.U = R * self.LyH
        self.L = -(-M // Ch) + (1 if W < Ch else 0)
        self.ring = list(range(P))
        self.start, self.free = 0, P
        self.table = [[-1] * self.L for _ in range(self.U)]
        self.sec = [{1: [], 2: []} for _ in range(self.U)]
        self.state = [IDLE] * R
        self.seq = [0] * R
        self.status = 0

    def _recycle(self):
        for r in range(self.R):
            if self.state[r] != PENDING:
                continue
            for u in range(r * self.LyH, (r + 1) * self.LyH):
                for k in range(self.L):
                    if self.table[u][k] != -1:
                        self.ring[(self.start + self.free) % self.P] = self.table[u][k]
                        self.free += 1
                        self.table[u][k] = -1
                self.sec[u] = {1: [], 2: []}
            self.state[r], self.seq[r] = IDLE, 0

    def _take(self, n):
        ids = [self.ring[(self.start + k) % self.P] for k in range(n)]
        self.start = (self.start + n) % self.P
        self.free -= n
        return ids

    def prefill_demand(self, reqs, lens, sig):
        """pages the admission would take, and the pages the same call recycles first (Q14)"""
        saved = (self.state[:], self.sec)
        D = 0
        for i, r in enumerate(reqs):
            n = lens[i]
            for j in range(self.LyH):
                nh = nl = 0
                for t in range(max(n - self.W, 0)):
                    s_ = f32(sig[i][j][t]) + f32(0)
                    if s_ >= self.ah / f32(t + 1):
                        nh += 1
                    elif s_ >= self.al / f32(t + 1):
                        nl += 1
                D += -(-nh // self.Ch) + -(-nl // self.Cl)
        rec = sum(1 for r in range(self.R) if self.state[r] == PENDING
                  for u in range(r * self.LyH, (r + 1) * self.LyH) for x in self.table[u] if x >= 0)
        self.state, self.sec = saved
        return D, rec

    def prefill(self, reqs, lens, sig):
        """sig[i][j][t]; the newest W tokens stay in the window (Q10)"""
        plans = {}
        for i, r in enumerate(reqs):
            n = lens[i]
            for j in range(self.LyH):
                u = r * self.LyH + j
                hi, lo = [], []
                for t in range(max(n - self.W, 0)):
                    s = f32(sig[i][j][t]) + f32(0)
                    th, tl = self.ah / f32(t + 1), self.al / f32(t + 1)        # §4, den = i (Q4 default)
                    if s >= th:
                        hi.append((s, t))
                    elif s >= tl:
                        lo.append((s, t))
                plans[u] = (hi, lo)
            self.state[r] = ADMITTING
        self._recycle()
        if self.status:
            return
        D = sum(-(-len(h) // self.Ch) + -(-len(l) // self.Cl) for h, l in plans.values())
        if D > self.free:
            self.status = oracle.ERR_OOM
            return
        for u in sorted(plans):                                   # canonical order (Q13)
            h, l = plans[u]
            ph, pl = -(-len(h) // self.Ch), -(-len(l) // self.Cl)
            ids = self._take(ph + pl)
            for k in range(ph):
                self.table[u][k] = ids[k]
            for k in range(pl):
                self.table[u][self.L - 1 - k] = ids[ph + k]
            self.sec[u] = {1: list(h), 2: list(l)}
        for i, r in enumerate(reqs):
            self.seq[r] = lens[i]
            self.state[r] = ACTIVE

    def decode(self, cand):
        self._recycle()
        if self.status:
            return
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
            th, tl = self.ah / f32(N), self.al / f32(N)
            if s >= th:
                cls, bar = 1, th
            elif s >= tl:
                cls, bar = 2, tl
            else:
                continue                                          # t_c pruned
            sec = self.sec[u][cls]
            cands = [(v, p, k) for k, (v, p) in enumerate(sec)] + [(s, pc, -1)]
            v, p, k = min(cands, key=lambda x: (x[0], x[1]))      # Q6: ties -> oldest
            if k == -1 or v >= bar:                               # t_v stays: t_c appended
                grows[u] = (cls, "append", (s, pc))
            elif cls == 1 and v >= tl:                            # downgrade t_v (Q8)
                grows[u] = (2, "down", (k, (s, pc), (v, p)))
            else:                                                 # prune t_v, t_c takes its slot
                grows[u] = (None, "replace", (cls, k, (s, pc)))
        demand = {}
        for u, (gcls, kind, _) in grows.items():
            if gcls is not None:
                n = len(self.sec[u][gcls])
                demand[u] = (n % (self.Ch if gcls == 1 else self.Cl) == 0)
        D = sum(demand.values())
        if D > self.free:
            self.status = oracle.ERR_OOM
            return
        for u in sorted(demand):
            if demand[u]:
                gcls = grows[u][0]
                n = len(self.sec[u][gcls])
                (pid,) = self._take(1)
                k = n // self.Ch if gcls == 1 else self.L - 1 - n // self.Cl
                self.table[u][k] = pid
        for u, (gcls, kind, x) in grows.items():
            if kind == "append":
                self.sec[u][gcls].append(x)
            elif kind == "down":
                k, tc, v = x
                self.sec[u][1][k] = tc
                self.sec[u][2].append(v)
            else:
                cls, k, tc = x
                self.sec[u][cls][k] = tc
        for r in range(self.R):
            if self.state[r] == ACTIVE:
                self.seq[r] += 1

    def free_req(self, reqs):
        for r in reqs:
            self.state[r] = PENDING


def _compare(m, pool, where):
    assert pool.status == m.status, where
    assert (pool.start, pool.free) == (m.start, m.free), where
    assert np.array_equal(pool.ring, np.array(m.ring, np.int32)), where
    assert np.array_equal(pool.table, np.array(m.table, np.int32).reshape(m.U, m.L)), where
    for u in range(m.U):
        for cls in (1, 2):
            n = int(pool.n_h[u] if cls == 1 else pool.n_l[u])
            assert n == len(m.sec[u][cls]), (where, u, cls)
            for s in range(n):
                _, _, _, _, sg, ps = pool.slot_record(cls, u, s)
                v, p = m.sec[u][cls][s]
                assert (sg, ps) == (int(np.float32(v).view(np.uint32)), p), (where, u, cls, s)
    # PIN-10 (I1): the free region and the tables hold every page exactly once
    ids = [m.ring[(m.start + k) % m.P] for k in range(m.free)] + [x for row in m.table for x in row if x >= 0]
    assert sorted(ids) == list(range(m.P)), where


def _lattice(rng, th, tl, size):
    vals = np.array([0.0, -0.0, tl, th, 2 * th, th / 2, tl / 2, (th + tl) / 2, 4 * th], np.float32)
    vals = vals[vals >= 0] if tl > 0 else vals
    return vals[rng.integers(0, len(vals), size=size)]


@pytest.mark.parametrize("Ch,W", [(1, 0), (1, 1), (2, 0), (2, 2), (4, 1)])
def test_bruteforce_tiny_lifecycles(Ch, W):
    rng = np.random.default_rng(100 * Ch + W)
    ah, al = 1.0, 0.25
    for case in range(200):
        R, Ly, H = int(rng.choice([1, 2, 3])), 1, int(rng.choice([1, 2]))
        if R * H > 3:
            H = 1
        P = int(rng.integers(4, 13))
        M = 12
        Cl = 2 * Ch
        cfg = oracle.make_config(R=R, Ly=Ly, H=H, d=8, M=M, W=W, Ch=Ch, Cl=Cl, P=P, alpha_h=ah, alpha_l=al)
        pool = oracle.OraclePool(cfg)
        m = Model(R, Ly, H, W, Ch, Cl, P, M, ah, al)
        U = R * Ly * H
        zeros_kv = lambda *shape: np.zeros(shape + (8,), np.float16)

        def admit(reqs):
            lens = [int(rng.integers(0, 7)) for _ in reqs]
            stride = max(max(lens), 1)
            sig = np.zeros((len(reqs), Ly * H, stride), np.float32)
            for t in range(stride):
                th, tl = f32(ah) / f32(t + 1), f32(al) / f32(t + 1)
                sig[:, :, t] = _lattice(rng, th, tl, (len(reqs), Ly * H))
            D, rec = m.prefill_demand(reqs, lens, sig)
            if D > m.free + rec:                                   # keep admissions within the pool
                return False
            st, _ = pool.classify_prefill(reqs, lens, sig)
            assert st == 0
            assert pool.compact_alloc(None) == 0
            k = zeros_kv(len(reqs), Ly * H, stride)
            assert pool.quant_write_prefill(k, k, sig) == 0
            m.prefill(reqs, lens, sig)
            assert m.status == 0
            return True

        live = [r for r in range(R) if admit([r])]
        _compare(m, pool, f"case {case} admit")
        for step in range(8):
            if any(m.seq[r] >= M for r in range(R) if m.state[r] == ACTIVE):
                break
            N = [m.seq[r] + 1 for r in range(R)]
            cand = np.zeros(U, np.float32)
            for u in range(U):
                n = f32(N[u // (Ly * H)])
                cand[u] = _lattice(rng, f32(ah) / n, f32(al) / n, 1)[0]
            st, dec = pool.classify_decode(cand)
            assert st == 0
            assert pool.compact_alloc(dec) == 0
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
                m.free_req(fr)
            idle = [r for r in range(R) if m.state[r] == IDLE]
            if idle and rng.random() < 0.3:
                admit([idle[0]])
                _compare(m, pool, f"case {case} re-admit {step}")
