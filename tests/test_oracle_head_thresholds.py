"""NEXT-4 pins (per-head thresholds, reading Q35): per-head thresholds equal to the pool-wide pair
reproduce the pool-wide run byte for byte (reduction); a head whose thresholds are raised beyond every
significance stores nothing while every other unit's sections stay exactly as in the pool-wide run; random
per-head thresholds keep the pool invariants (PIN-10) after every call; invalid values are rejected."""
import numpy as np
import pytest

import oracle
from tests import harness as H


def _run(scn, head=None, steps=24, inp_scn=None):
    o = H.OracleBackend(scn)
    if head is not None:
        assert o.pool.set_head_thresholds(*head) == 0
    inp, life = H.Inputs(inp_scn or scn), H.Lifecycle(scn)
    H.admit([o], inp, life, list(range(scn.R)), [60 + 11 * r for r in range(scn.R)])
    H.check_invariants(o.snapshot(), scn, o.L, o.geom, life if head is None else None)
    for step in range(steps):
        H.decode_step([o], inp, life, step)
        H.check_invariants(o.snapshot(), scn, o.L, o.geom, life if head is None else None)
    return o


SCN = H.TINY.replace(R=3, Ly=2, H=3, d=64, M=160, W=8, Ch=8, Cl=16, P=3000, seed=31)


def test_uniform_head_thresholds_reduce_to_pool_wide():
    n = SCN.Ly * SCN.H
    a = _run(SCN)
    b = _run(SCN, head=(np.full(n, SCN.alpha_h, np.float32), np.full(n, SCN.alpha_l, np.float32)))
    sa, sb = a.snapshot(), b.snapshot()
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), k


def _records(o, u):
    p = o.pool
    out = []
    for cls, n in ((1, p.n_h[u]), (2, p.n_l[u])):
        for s in range(int(n)):
            kc, km, vc, vm, sg, ps = p.slot_record(cls, u, s)
            out.append((cls, s, bytes(kc), km, bytes(vc), vm, sg, ps))
    return out


def test_silenced_head_stores_nothing_and_others_are_unchanged():
    n = SCN.Ly * SCN.H
    ah = np.full(n, SCN.alpha_h, np.float32)
    al = np.full(n, SCN.alpha_l, np.float32)
    quiet = 4                                                   # (layer 1, head 1)
    ah[quiet], al[quiet] = 1e30, 1e30                           # every token below alpha_l / i: pruned
    a = _run(SCN)
    b = _run(SCN, head=(ah, al))
    for u in range(SCN.U):
        if u % n == quiet:
            assert b.pool.n_h[u] == 0 and b.pool.n_l[u] == 0 and (b.pool.table[u] == -1).all()
        else:
            assert _records(a, u) == _records(b, u), u


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_head_thresholds_keep_invariants(seed):
    rng = np.random.default_rng(seed)
    n = SCN.Ly * SCN.H
    ah = rng.choice([0.5, 1.0, 3.0], size=n).astype(np.float32)
    al = rng.choice([0.0, 0.02, 0.1], size=n).astype(np.float32)
    o = _run(SCN.replace(seed=seed), head=(ah, al), steps=30, inp_scn=SCN.replace(seed=seed))
    assert o.pool.status == 0


def test_invalid_head_thresholds_rejected():
    o = H.OracleBackend(SCN)
    n = SCN.Ly * SCN.H
    bad = np.full(n, 1.0, np.float32)
    bad[2] = np.nan
    assert o.pool.set_head_thresholds(bad, np.zeros(n, np.float32)) == oracle.ERR_INVALID
    bad[2] = -1.0
    assert o.pool.set_head_thresholds(np.ones(n, np.float32), bad) == oracle.ERR_INVALID
    assert o.pool.set_head_thresholds(None, None) == 0
