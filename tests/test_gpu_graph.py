"""The decode step as a CUDA graph (dkv_decode_graph_*): replaying a captured graph —
with programmatic dependent launch between its kernels, with per-kernel event nodes, or plain — gives the
same decisions and pool state, byte for byte, as the eager calls and the oracle, across a free (recycled by
the graph's first step, its page copies done by that step's quant_write kernel) and a re-admission made with
eager calls between graph launches; a graph of several steps replays several steps."""
import numpy as np
import pytest
import torch

from tests import harness as H

pytestmark = pytest.mark.gpu


def _backends(scn):
    from tests.gpu_backend import GpuBackend
    return H.OracleBackend(scn), GpuBackend(scn)


def _check(o, g, where, do=None, dg=None):
    from tests.gpu_backend import compare_state, dec_np
    if do is not None:
        a, b = dec_np(do), dec_np(dg)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"[{where}] decisions differ"
    compare_state(o.snapshot(), g.snapshot(), where=where)
    assert g.snapshot(pages=False)["status"] == 0


@pytest.mark.parametrize("flags", [0, 1, 2], ids=["plain", "pdl", "events"])
def test_graph_single_step_replay_matches_oracle(flags):
    from paper_2412_03131_b200 import dkv as D
    scn = H.TINY.replace(R=6, Ly=2, H=4, d=64, M=256, W=16, P=6000, seed=51, tile_units=256)
    o, g = _backends(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, list(range(scn.R)), [70, 33, 120, 16, 90, 64])
    dev = g.device
    sig = torch.zeros(scn.U, dtype=torch.float32, device=dev)
    k = torch.zeros((scn.U, scn.d), dtype=torch.int16, device=dev)
    v = torch.zeros_like(k)
    dec = g.pool.new_decisions()
    graph = g.pool.decode_graph(1, sig, k, v, dec, flags)
    for step in range(36):
        o.drift(step)
        g.drift(step)
        active = life.state == H.REQ_ACTIVE
        N = np.where(active, life.seq + 1, 0)
        cand, kk, vv = inp.decode(N)
        st, do = o.classify_decode(cand)
        assert st == 0 and o.compact_alloc(do) == 0 and o.quant_write_decode(do, kk, vv, cand) == 0
        sig.copy_(cand.to(dev))
        k.copy_(kk.to(dev).view(torch.int16))
        v.copy_(vv.to(dev).view(torch.int16))
        graph.launch()
        torch.cuda.synchronize()
        life.seq[active] += 1
        _check(o, g, f"step {step}", do, dec)
        if flags & D.DKV_GRAPH_EVENTS:
            ms = graph.kernel_ms()
            assert (ms > 0).all() and (ms < 50).all(), ms
        if step == 9:
            H.free([o, g], life, [2, 4])                       # recycled by the next graph launch
        if step == 15:
            H.admit([o, g], inp, life, [2], [100])             # eager calls between graph launches
            _check(o, g, "re-admitted")
    st, _ = g.pool.query()
    assert st == 0
    graph.close()


def test_graph_of_several_steps_replays_them():
    """8 steps in one graph (per-step input buffers, PDL): the state after one launch equals 8 oracle steps;
    then a free and a second launch whose first step recycles the request."""
    from paper_2412_03131_b200 import dkv as D
    scn = H.TINY.replace(R=5, Ly=3, H=4, d=128, M=400, W=64, P=9000, seed=52)
    o, g = _backends(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, list(range(scn.R)), [200, 64, 150, 99, 70])
    T = 8
    dev = g.device
    sig = torch.zeros((T, scn.U), dtype=torch.float32, device=dev)
    k = torch.zeros((T, scn.U, scn.d), dtype=torch.int16, device=dev)
    v = torch.zeros_like(k)
    dec = g.pool.new_decisions()
    graph = g.pool.decode_graph(T, sig, k, v, dec, D.DKV_GRAPH_PDL)
    for launch in range(2):
        do = None
        for t in range(T):
            active = life.state == H.REQ_ACTIVE
            N = np.where(active, life.seq + 1, 0)
            cand, kk, vv = inp.decode(N)
            st, do = o.classify_decode(cand)
            assert st == 0 and o.compact_alloc(do) == 0 and o.quant_write_decode(do, kk, vv, cand) == 0
            life.seq[active] += 1
            life.state[life.state == H.REQ_PENDING_FREE] = H.REQ_IDLE
            sig[t].copy_(cand.to(dev))
            k[t].copy_(kk.to(dev).view(torch.int16))
            v[t].copy_(vv.to(dev).view(torch.int16))
        graph.launch()
        torch.cuda.synchronize()
        _check(o, g, f"launch {launch}", do, dec)               # the last step's decisions
        if launch == 0:
            H.free([o, g], life, [1, 3])
    graph.close()


def test_graph_launch_checks_lengths():
    """a launch whose steps would take an ACTIVE request past max_seq_len is refused before anything runs"""
    from paper_2412_03131_b200 import dkv as D
    scn = H.TINY.replace(R=2, Ly=1, H=2, d=64, M=80, W=16, P=500)
    o, g = _backends(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([g], inp, life, [0, 1], [70, 40])
    T = 12
    sig = torch.zeros((T, scn.U), dtype=torch.float32, device=g.device)
    k = torch.zeros((T, scn.U, scn.d), dtype=torch.int16, device=g.device)
    graph = g.pool.decode_graph(T, sig, k, k.clone(), g.pool.new_decisions(), D.DKV_GRAPH_PDL)
    with pytest.raises(RuntimeError):
        graph.launch()                                          # 70 + 12 > 80
    H.free([g], life, [0])
    graph2 = g.pool.decode_graph(1, sig[0], k[0], k[0].clone(), g.pool.new_decisions(), 0)
    graph2.launch()
    graph.launch()                                              # request 1: 41 + 12 <= 80
    torch.cuda.synchronize()
    st, _ = g.pool.query()
    assert st == 0
