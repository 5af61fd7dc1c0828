"""NEXT-1 pins: the paper's prompt-phase workflow (fig:memory_management_flow) in the oracle,
selected by prefill_workflow = 1 — conservative allocation of ceil(kept/C_h) pages per head, planning,
keep high pages from the left and low pages from the right, reclaim the middle at the end pointer (one
top-up page when the plan needs it, reading Q29).

Pinned against: the paper's worked example (Fig. 5, tests/golden/fig5.json) at its own geometry and
scaled to 4-token high pages; the exact-allocation workflow, which must store identical section contents
(classes, counts, codes, metadata, scores, positions — only page IDs differ); the pool invariants
(PIN-10); and a small independent model of the ring/table steps as the paper's text orders them."""
import json
import os

import numpy as np
import pytest

import oracle
from tests import harness as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _fig5():
    with open(os.path.join(GOLD, "fig5.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("scale", [1, 2])
def test_fig5_through_compact_alloc(scale):
    """Fig. 5 via the regular call sequence (classify(PREFILL) -> compact_alloc) with prefill_workflow = 1;
    scale 2 doubles the tokens per page and repeats every token (the GPU geometry needs C % 4 == 0)."""
    g = _fig5()
    c = dict(g["config"])
    c.update(Ch=c["Ch"] * scale, Cl=c["Cl"] * scale, M=c["M"] * scale, prefill_workflow=1)
    pool = oracle.OraclePool(oracle.make_config(**c))
    pool.start, pool.free = g["initial"]["start"], g["initial"]["free"]
    n = g["prompt_len"] * scale
    sig = np.repeat(np.array(g["sig"], np.float32), scale, axis=1).reshape(1, 2, n)
    # significance scales with 1/i under alpha/i (Q4): rescale so every token keeps its Fig. 5 class
    if scale > 1:
        i = np.arange(1, n + 1, dtype=np.float32)
        base = np.repeat(np.arange(1, g["prompt_len"] + 1, dtype=np.float32), scale)
        sig = (sig * (base / i)).astype(np.float32)
    st, cls = pool.classify_prefill([0], [n], sig)
    assert st == 0
    assert pool.compact_alloc(None) == 0 and pool.status == oracle.OK
    e = g["expect"]
    L = pool.L
    for head, u in (("A", 0), ("B", 1)):
        row = pool.table[u]
        assert list(row[:len(e["high_pages"][head])]) == e["high_pages"][head]
        assert [int(row[L - 1 - k]) for k in range(len(e["low_pages"][head]))] == e["low_pages"][head]
    assert list(pool.ring[:3]) == e["ring_head_after"]
    assert pool.start == e["start_after"] and pool.free == e["free_after"]
    assert pool.last_reclaimed == len(e["reclaimed_in_order"])


def test_topup_page_when_plan_exceeds_block():
    """Q29: one High and one Low token in a 4-token block -> ceil(1/4) + ceil(1/8) = 2 > 1 page: the head
    keeps its block page for High and takes the top-up page (granted after every block) for Low."""
    pool = oracle.OraclePool(oracle.make_config(R=1, Ly=1, H=2, d=64, M=8, W=0, Ch=4, Cl=8, P=16,
                                                alpha_h=1.0, alpha_l=0.02, prefill_workflow=1))
    # unit 0: tokens H, L (kept 2 -> block of 1 page, plan 1 + 1); unit 1: H, H (block 1, plan 1, no reclaim)
    sig = np.array([[[2.0, 0.05], [2.0, 2.0]]], np.float32)
    st, _ = pool.classify_prefill([0], [2], sig)
    assert st == 0 and pool.compact_alloc(None) == 0 and pool.status == oracle.OK
    L = pool.L
    # blocks: unit 0 -> page 0, unit 1 -> page 1; top-up for unit 0 -> page 2 (after all blocks)
    assert pool.table[0, 0] == 0 and pool.table[0, L - 1] == 2
    assert pool.table[1, 0] == 1 and (pool.table[1, 1:] == -1).all()
    assert pool.start == 3 and pool.free == 13 and pool.last_reclaimed == 0 and pool.last_demand == 3


class PaperWorkflowModel:
    """The prompt workflow as the paper's text orders it plus Q29, on ring / table only:
    blocks from the allocation pointer in canonical head order, then top-ups, then the kept pages go left
    (high) / right (low) and the middles are appended at the end pointer, head by head."""

    def __init__(self, P, start, free, L):
        self.ring = list(range(P))
        self.P, self.start, self.free, self.L = P, start, free, L

    def prompt(self, blocks, plans):
        P = self.P
        end = (self.start + self.free) % P
        need = [(ph + pl > c) for c, (ph, pl) in zip(blocks, plans)]
        D = sum(blocks) + sum(need)
        if D > self.free:
            return None
        pos = self.start
        got = []
        for c in blocks:
            got.append([self.ring[(pos + k) % P] for k in range(c)])
            pos += c
        for i, n in enumerate(need):
            if n:
                got[i].append(self.ring[pos % P])
                pos += 1
        tables = []
        reclaimed = []
        for blk, (ph, pl) in zip(got, plans):
            row = [-1] * self.L
            for k in range(ph):
                row[k] = blk[k]
            for k in range(pl):
                row[self.L - 1 - k] = blk[len(blk) - 1 - k]
            reclaimed += blk[ph:len(blk) - pl]
            tables.append(row)
        for k, pid in enumerate(reclaimed):
            self.ring[(end + k) % P] = pid
        self.start = (self.start + D) % P
        self.free = self.free - D + len(reclaimed)
        return tables


@pytest.mark.parametrize("seed", range(40))
def test_oracle_matches_paper_workflow_model(seed):
    rng = np.random.default_rng(seed)
    Ch = int(rng.choice([4, 8]))
    Cl = Ch * int(rng.choice([1, 2]))
    H_, W = int(rng.integers(1, 4)), int(rng.choice([0, 4]))
    M = 48
    P = int(rng.integers(8, 64))
    cfg = oracle.make_config(R=2, Ly=1, H=H_, d=64, M=M, W=W, Ch=Ch, Cl=Cl, P=P, alpha_h=1.0, alpha_l=0.02,
                             prefill_workflow=1)
    pool = oracle.OraclePool(cfg)
    pool.start = int(rng.integers(0, P))
    model = PaperWorkflowModel(P, pool.start, pool.free, pool.L)
    n = int(rng.integers(0, M + 1))
    i = np.arange(1, n + 1, dtype=np.float32)
    pick = rng.integers(0, 3, size=(1, H_, n))
    sig = np.where(pick == 0, 2.0 / i, np.where(pick == 1, 0.1 / i, 0.001 / i)).astype(np.float32)
    st, cls = pool.classify_prefill([0], [n], sig)
    assert st == 0
    kept = max(n - W, 0)
    plans = [(H.ceil_div(int((cls[0, h, :kept] == 1).sum()), Ch), H.ceil_div(int((cls[0, h, :kept] == 2).sum()), Cl))
             for h in range(H_)]
    blocks = [H.ceil_div(kept, Ch)] * H_
    tables = model.prompt(blocks, plans)
    assert pool.compact_alloc(None) == 0
    if tables is None:
        assert pool.status == oracle.ERR_OOM
        return
    assert pool.status == oracle.OK
    assert np.array_equal(pool.table[:H_], np.array(tables, np.int32).reshape(H_, pool.L))
    assert np.array_equal(pool.ring, np.array(model.ring, np.int32))
    assert (pool.start, pool.free) == (model.start, model.free)


def _lifecycle(scn, steps=24, frees=((9, [1]),)):
    o = H.OracleBackend(scn)
    inp = H.Inputs(scn)
    life = H.Lifecycle(scn)
    H.admit([o], inp, life, list(range(scn.R)), [64 + 7 * r for r in range(scn.R)])
    snaps = [o.snapshot()]
    H.check_invariants(snaps[-1], scn, o.L, o.geom, life)
    for step in range(steps):
        H.decode_step([o], inp, life, step)
        H.check_invariants(o.snapshot(), scn, o.L, o.geom, life)
        for t, rs in frees:
            if step == t:
                H.free([o], life, rs)
                H.decode_step([o], inp, life, 1000 + step)     # recycles
                H.admit([o], inp, life, rs, [50] * len(rs))
                H.check_invariants(o.snapshot(), scn, o.L, o.geom, life)
    return o


def _section_records(o):
    out = []
    p = o.pool
    for u in range(p.U):
        for cls, n in ((1, p.n_h[u]), (2, p.n_l[u])):
            for s in range(int(n)):
                kc, km, vc, vm, sg, ps = p.slot_record(cls, u, s)
                out.append((u, cls, s, bytes(kc), km, bytes(vc), vm, sg, ps))
    return out


@pytest.mark.parametrize("mix", [(0.35, 0.45, 0.20), (0.05, 0.90, 0.05), (0.6, 0.1, 0.3)])
def test_workflows_store_identical_sections(mix):
    """Both prompt workflows apply the same plan: identical counts, decisions and per-slot
    records (codes, metadata, score, position) through prefill, decode and re-admission; the pages used
    equal sum(ceil(n_h/C_h) + ceil(n_l/C_l)) either way."""
    base = H.TINY.replace(R=3, Ly=2, H=3, d=64, M=160, W=8, Ch=8, Cl=16, P=4000, mix=mix, seed=17)
    a = _lifecycle(base.replace(prefill_workflow=0))
    b = _lifecycle(base.replace(prefill_workflow=1))
    assert np.array_equal(a.pool.n_h, b.pool.n_h) and np.array_equal(a.pool.n_l, b.pool.n_l)
    assert a.pool.free == b.pool.free
    assert _section_records(a) == _section_records(b)
