"""dkv_audit (the SURVEY's debug audit kernel): the pool's invariants checked on the device — every page owned once
(free region or one occupied slot), occupied slots exactly the [0, ceil(n_h/C_h)) / [L - ceil(n_l/C_l), L) ranges
(P:495-499), every other slot empty, stored positions unique and below N - W — clean on sound pools after a
lifecycle with frees and re-admission (both prompt workflows, the three-level tier), and each kind of corruption
planted in a pool's state is reported."""
import numpy as np
import pytest
import torch

from tests import harness as H

pytestmark = pytest.mark.gpu

CLEAN = ("owned_twice", "unowned", "bad_slots", "dup_positions", "positions_out_of_range", "over_capacity")


def _lifecycle(scn, steps=10):
    from tests.gpu_backend import GpuBackend
    g = GpuBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([g], inp, life, list(range(scn.R)), [int(x) for x in np.linspace(40, scn.M // 2, scn.R)])
    for step in range(steps):
        H.decode_step([g], inp, life, step)
        if step == steps // 2:
            H.free([g], life, [1])
    H.decode_step([g], inp, life, steps)                       # recycles the freed request
    life.state[life.state == H.REQ_PENDING_FREE] = H.REQ_IDLE
    H.admit([g], inp, life, [1], [scn.M // 3])
    return g


def _sound(g, P):
    a = g.pool.audit()
    assert a["used_pages"] + a["free_pages"] == P, a
    assert all(a[k] == 0 for k in CLEAN), a
    return a


@pytest.mark.parametrize("kw", [dict(), dict(prefill_workflow=1), dict(tile_units=256),
                                dict(top_tier=1, alpha_t=2.0, Ct=4)])
def test_audit_clean_after_lifecycle(kw):
    scn = H.TINY.replace(R=6, Ly=2, H=3, d=64, M=600, W=16, P=5000, seed=17, **kw)
    g = _lifecycle(scn)
    a = _sound(g, scn.P)
    assert a["used_pages"] > 0


def test_audit_reports_planted_corruption():
    scn = H.TINY.replace(R=6, Ly=2, H=3, d=64, M=600, W=16, P=5000, seed=19)
    g = _lifecycle(scn, steps=4)
    _sound(g, scn.P)
    v = g.pool.views()
    table, n_h = v["table"], v["n_h"].cpu().numpy()
    L = g.L
    us = [u for u in range(g.U) if n_h[u] >= 1]
    u0, u1 = us[0], us[1]
    torch.cuda.synchronize()
    saved = table[u0, 0].item()
    table[u0, 0] = table[u1, 0]                                # a page owned twice, another owned by nobody
    torch.cuda.synchronize()
    a = g.pool.audit()
    assert a["owned_twice"] == 1 and a["unowned"] == 1, a
    table[u0, 0] = saved
    ph = -(-int(n_h[u0]) // scn.Ch)
    table[u0, ph] = 3                                          # an unoccupied slot that is not empty (its stray
    torch.cuda.synchronize()                                   # ID is not an owner: the page stays owned once)
    a = g.pool.audit()
    assert a["bad_slots"] == 1 and a["owned_twice"] == 0 and a["unowned"] == 0, a
    table[u0, ph] = -1
    torch.cuda.synchronize()
    _sound(g, scn.P)
    # a duplicated stored position: copy the position of high slot 0 into high slot 1 of the same unit
    u = [x for x in range(g.U) if n_h[x] >= 2][0]
    geo = g.geom[1]
    pid = int(table[u, 0].item())
    pages = v["pages"]
    p0 = pages[pid, geo["off_pos"]: geo["off_pos"] + 4].clone()
    keep = pages[pid, geo["off_pos"] + 4: geo["off_pos"] + 8].clone()
    pages[pid, geo["off_pos"] + 4: geo["off_pos"] + 8] = p0
    torch.cuda.synchronize()
    a = g.pool.audit()
    assert a["dup_positions"] == 1, a
    pages[pid, geo["off_pos"] + 4: geo["off_pos"] + 8] = keep
    torch.cuda.synchronize()
    _sound(g, scn.P)


def test_audit_requires_idle_pool():
    from paper_2412_03131_b200 import dkv as D
    g = _lifecycle(H.TINY.replace(R=4), steps=2)
    g.pool.classify_decode(torch.zeros(g.U, device="cuda"), g.dec)   # mid-step: the call is refused
    with pytest.raises(D.DkvError):
        g.pool.audit()
