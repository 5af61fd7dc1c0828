"""Test / bench harness: scenarios, seeded inputs for both sides, a lifecycle driver, and the state
invariants the paper fixes (PIN-10).  Holds none of the method's arithmetic.

A *backend* is anything with the methods below; ``OracleBackend`` wraps the serial oracle and
``tests/gpu_backend.py`` wraps the CUDA C-ABI.  The driver feeds both the same synth inputs.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np
import torch

import synth

REQ_IDLE, REQ_ADMITTING, REQ_ACTIVE, REQ_PENDING_FREE = 0, 1, 2, 3


@dataclass
class Scenario:
    R: int = 4
    Ly: int = 2
    H: int = 4
    d: int = 64
    M: int = 128
    W: int = 16
    Ch: int = 16
    Cl: int = 32
    kbh: int = 8
    vbh: int = 4
    kbl: int = 4
    vbl: int = 2
    P: int = 1024
    alpha_h: float = 1.0
    alpha_l: float = 0.02
    prompt_denominator: int = 0
    prefill_workflow: int = 0
    q_per_kv: int = 0
    seed: int = 1
    mix: tuple = (0.35, 0.45, 0.20)
    H_total: int | None = None
    h0: int = 0
    tile_units: int = 0
    req_ids: tuple | None = None      # global request ids of the local slots (sampled sub-pools)
    top_tier: int = 0                 # NEXT-4: FP16 tier above K8V4 (Q38-Q44)
    alpha_t: float = 0.0
    Ct: int = 4

    @property
    def shape(self) -> synth.Shape:
        return synth.Shape(self.R, self.Ly, self.H, self.H_total, self.h0, self.req_ids)

    @property
    def U(self):
        return self.R * self.Ly * self.H

    @property
    def LyH(self):
        return self.Ly * self.H

    def config_dict(self):
        return {k: getattr(self, k) for k in ("R", "Ly", "H", "d", "M", "W", "Ch", "Cl", "kbh", "vbh", "kbl", "vbl",
                                              "P", "alpha_h", "alpha_l", "prompt_denominator",
                                              "prefill_workflow", "q_per_kv", "top_tier", "alpha_t", "Ct")}

    def replace(self, **kw):
        return dataclasses.replace(self, **kw)


TINY = Scenario()   # BASELINE.json configs[0]: 4 req x 2 layers x 4 heads, d 64, 64 tokens, 16-token pages, 1024 pages


# ------------------------------------------------------------------------------------------ inputs
class Inputs:
    """Seeded inputs for a scenario; every tensor is produced on `device` from counters only."""

    def __init__(self, scn: Scenario, device="cpu"):
        self.scn = scn
        self.device = device
        ug = scn.shape.global_units(list(range(scn.R)), device="cpu")         # [R, LyH]
        self.ug = ug.to(device)
        mh, ml = synth.unit_mix(scn.seed, ug, scn.mix, Ly=scn.Ly, Ht=scn.shape.Ht)
        self.mix_h, self.mix_l = mh.to(device), ml.to(device)

    def prefill(self, reqs, lens, stride=None):
        s = self.scn
        stride = int(stride if stride is not None else max(max(lens, default=0), 1))
        ridx = torch.as_tensor(np.asarray(reqs, np.int64), device=self.device)
        ug = self.ug[ridx]                                                         # [n, LyH]
        sig = synth.prefill_sig(s.seed, ug, stride, s.alpha_h, s.alpha_l, self.mix_h[ridx], self.mix_l[ridx],
                                lens=lens, denominator=s.prompt_denominator)
        k = synth.kv_values(s.seed, synth.S_KEY, ug, 0, stride, s.d)
        v = synth.kv_values(s.seed, synth.S_VAL, ug, 0, stride, s.d)
        return sig, k, v

    def decode(self, N_req):
        """N_req: int64 [R] request length INCLUDING the token appended this step (0 = not active)."""
        s = self.scn
        N = torch.as_tensor(np.asarray(N_req, np.int64), device=self.device).view(-1, 1).expand(-1, s.LyH).reshape(-1)
        ug = self.ug.reshape(-1)
        cand = synth.decode_sig(s.seed, ug, N, s.W, s.alpha_h, s.alpha_l, self.mix_h.reshape(-1), self.mix_l.reshape(-1))
        k, v = synth.new_token_kv(s.seed, ug, (N - 1).clamp(min=0), s.d)
        return cand, k, v


# ------------------------------------------------------------------------------------------ oracle backend
class OracleBackend:
    name = "oracle"

    def __init__(self, scn: Scenario):
        import oracle
        self.o = oracle
        self.scn = scn
        self.pool = oracle.OraclePool(oracle.make_config(**scn.config_dict()))
        self.U, self.L, self.page_bytes = self.pool.U, self.pool.L, self.pool.page_bytes
        g = self.pool.geom
        self.geom = {c: dict(C=g[c].C, k_row=g[c].k_row, v_row=g[c].v_row, off_k=g[c].off_k,
                             off_kmeta=g[c].off_kmeta, off_v=g[c].off_v, off_vmeta=g[c].off_vmeta,
                             off_score=g[c].off_score, off_pos=g[c].off_pos) for c in g}

    def classify_decode(self, cand):
        return self.pool.classify_decode(None if cand is None else _np(cand))

    def classify_prefill(self, reqs, lens, sig):
        st, _ = self.pool.classify_prefill(reqs, lens, _np(sig), want_classes=False)
        return st

    def compact_alloc(self, dec):
        return self.pool.compact_alloc(None if dec is None else _np(dec))

    def quant_write_decode(self, dec, k, v, cand):
        return self.pool.quant_write_decode(_np(dec), _np(k), _np(v), None if cand is None else _np(cand))

    def attend(self, q, want_out=True, want_probs=False):
        return self.pool.attend(q, want_out=want_out, want_probs=want_probs)

    def set_head_thresholds(self, ah, al):
        return self.pool.set_head_thresholds(ah, al)

    def quant_write_prefill(self, k, v, sig):
        return self.pool.quant_write_prefill(_np(k), _np(v), _np(sig))

    def free(self, reqs):
        return self.pool.free_requests(reqs)

    def take_status(self):
        return self.pool.take_status()

    def drift(self, step):
        p = self.pool
        top = self.scn.top_tier
        synth.apply_drift(self.scn.seed, step, self.scn.shape, torch.from_numpy(p.pages),
                          torch.from_numpy(p.table), torch.from_numpy(p.n_h), torch.from_numpy(p.n_l),
                          {c: (self.geom[c]["C"], self.geom[c]["off_score"], self.geom[c]["off_pos"]) for c in self.geom},
                          self.L, ttable=torch.from_numpy(p.ttable) if top else None,
                          n_t=torch.from_numpy(p.n_t) if top else None)

    def snapshot(self, pages=True):
        p = self.pool
        s = dict(ring=p.ring.copy(), start=int(p.start), free=int(p.free), table=p.table.copy(),
                 n_h=p.n_h.copy(), n_l=p.n_l.copy(), req_state=p.req_state.copy(), seq_len=p.seq_len.copy(),
                 win_k=p.win_k.copy(), win_v=p.win_v.copy(), win_sig=p.win_sig.copy())
        if self.scn.top_tier:
            s.update(ttable=p.ttable.copy(), n_t=p.n_t.copy())
        if pages:
            s["pages"] = p.pages.copy()
        return s


def _np(x):
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu()
        if x.dtype == torch.float16:
            return x.view(torch.int16).numpy().view(np.uint16)
        return x.numpy()
    return x


# ------------------------------------------------------------------------------------------ driver
@dataclass
class Lifecycle:
    """Host-side bookkeeping of request lengths and of per-unit pruned counts (for invariant I4)."""
    scn: Scenario
    seq: np.ndarray = None
    pruned: np.ndarray = None
    state: np.ndarray = None

    def __post_init__(self):
        self.seq = np.zeros(self.scn.R, np.int64)
        self.pruned = np.zeros(self.scn.U, np.int64)
        self.state = np.zeros(self.scn.R, np.int8)


def admit(backends, inp: Inputs, life: Lifecycle, reqs, lens, check=None):
    scn = inp.scn
    sig, k, v = inp.prefill(reqs, lens)
    for b in backends:
        assert b.classify_prefill(reqs, lens, sig) == 0
    if check: check("classify_prefill")
    for b in backends:
        assert b.compact_alloc(None) == 0
    if check: check("compact_alloc_prefill")
    for b in backends:
        assert b.quant_write_prefill(k, v, sig) == 0
    if check: check("quant_write_prefill")
    # host bookkeeping of pruned prompt tokens (only used by invariant I4): §4 thresholds restated
    sg = _np(sig)
    scn = life.scn                                   # the pool's thresholds (inputs may be drawn for others)
    ah, al = np.float32(scn.alpha_h), np.float32(scn.alpha_l)
    for i, r in enumerate(reqs):
        T = int(lens[i])
        kept = max(T - scn.W, 0)
        den = (np.arange(kept) + 1).astype(np.float32) if scn.prompt_denominator == 0 else np.full(kept, T, np.float32)
        s = sg[i, :, :kept]
        life.pruned[r * scn.LyH:(r + 1) * scn.LyH] = (s < (al / den)[None, :]).sum(axis=1)
        life.seq[r] = T
        life.state[r] = REQ_ACTIVE
    return sig


def decode_step(backends, inp: Inputs, life: Lifecycle, step: int, check=None, drift=True):
    scn = inp.scn
    if drift:
        for b in backends:
            b.drift(step)
        if check: check("drift")
    active = life.state == REQ_ACTIVE
    N = np.where(active, life.seq + 1, 0)
    cand, k, v = inp.decode(N)
    decs = []
    for b in backends:
        st, dec = b.classify_decode(cand)
        assert st == 0
        decs.append(dec)
    if check: check("classify_decode", decs=decs)
    for b, dec in zip(backends, decs):
        assert b.compact_alloc(dec) == 0
    if check: check("compact_alloc", decs=decs)
    for b, dec in zip(backends, decs):
        assert b.quant_write_decode(dec, k, v, cand) == 0
    if check: check("quant_write_decode", decs=decs)
    life.seq[active] += 1
    d0 = _np(decs[0])
    if d0.dtype.names is None:                       # CUDA decisions: int32 [U, 4] -> 16-byte records
        import oracle
        d0 = np.ascontiguousarray(d0).view(oracle.DECISION_DTYPE).reshape(-1)
    pr =(d0["tc_class"] == 3).astype(np.int64) + (d0["v_action"] == 3).astype(np.int64)
    life.pruned += pr
    return decs


def free(backends, life: Lifecycle, reqs):
    for b in backends:
        assert b.free(reqs) == 0
    for r in reqs:
        life.state[r] = REQ_PENDING_FREE


# ------------------------------------------------------------------------------------------ invariants
def ceil_div(a, b):
    return -(-a // b)


def check_invariants(snap, scn: Scenario, L: int, geom, life: Lifecycle | None = None, prefill_pruned=None):
    """PIN-10: (I1) ring free region + table entries = {0..P-1} exactly once; (I2) occupied slots are
    exactly [0, ph) u [L-pl, L); (I3) stored positions unique per unit, all < N - W; (I4) stored + window +
    pruned = N (when the lifecycle tracks pruned counts)."""
    P = scn.P
    ring, start, free = snap["ring"], snap["start"], snap["free"]
    table, n_h, n_l = snap["table"], snap["n_h"], snap["n_l"]
    assert 0 <= free <= P and 0 <= start < P
    free_ids = ring[(start + np.arange(free)) % P]
    used = table[table >= 0]
    if "ttable" in snap:                              # NEXT-4: the TOP table's pages, slots [0, pt) occupied
        tt = snap["ttable"]
        used = np.concatenate([used, tt[tt >= 0]])
        pt = ceil_div(snap["n_t"], scn.Ct)
        assert np.array_equal(tt >= 0, np.arange(tt.shape[1])[None, :] < pt[:, None]), "TOP slots not [0, pt)"
    allids = np.concatenate([free_ids, used])
    assert allids.size == P, f"used + free = {allids.size} != P = {P}"
    assert np.array_equal(np.sort(allids), np.arange(P)), "a page is owned twice or lost"
    ph = ceil_div(n_h, scn.Ch)
    pl = ceil_div(n_l, scn.Cl)
    assert (ph + pl <= L).all()
    k = np.arange(L)[None, :]
    expect = (k < ph[:, None]) | (k >= (L - pl)[:, None])
    assert np.array_equal(table >= 0, expect), "occupied slots are not [0,ph) u [L-pl,L)"
    if "pages" in snap and life is not None:
        pages = snap["pages"]
        LyH = scn.LyH
        for u in range(scn.U):
            r = u // LyH
            if snap["req_state"][r] not in (REQ_ACTIVE, REQ_PENDING_FREE):
                continue
            N = int(snap["seq_len"][r])
            poss = []
            secs = ((1, n_h[u]), (2, n_l[u])) + (((4, snap["n_t"][u]),) if "ttable" in snap else ())
            for cls, n in secs:
                g = geom[cls]
                for s in range(int(n)):
                    if cls == 4:
                        pid = snap["ttable"][u, s // g["C"]]
                    else:
                        kk = s // g["C"] if cls == 1 else L - 1 - s // g["C"]
                        pid = table[u, kk]
                    idx = s % g["C"]
                    poss.append(int(pages[pid, g["off_pos"] + 4 * idx: g["off_pos"] + 4 * idx + 4].view("<i4")[0]))
            poss = np.array(poss, np.int64)
            assert len(np.unique(poss)) == len(poss), f"unit {u}: duplicate stored position"
            assert (poss < max(N - scn.W, 0)).all() and (poss >= 0).all()
            if life is not None and life.pruned is not None:
                nt = int(snap["n_t"][u]) if "n_t" in snap else 0
                assert int(n_h[u] + n_l[u]) + nt + min(scn.W, N) + int(life.pruned[u]) == N, f"I4 fails at unit {u}"
