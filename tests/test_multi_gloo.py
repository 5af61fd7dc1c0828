"""Multi-GPU path on CPU (gloo, world_size 2): KV heads sharded over ranks with one independent pool per
rank, the per-step MIN all-reduce of the admission counters, and PIN-13: every global unit's
logical content (classes, codes, metadata, scores, positions) is identical whether its heads live on one
pool or are sharded over two.  The pools here are oracle pools (the CUDA pools are per-GPU and never
exchange KV bytes; only the counters cross ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_03131_b200.admission import Admission, count_allreduce, prefill_page_bound, shard_heads
from tests import harness as H


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _unit_contents(backend, scn):
    """global unit id -> tuple of per-slot records sorted by position (page IDs excluded by design)."""
    o = backend.pool
    ug = scn.shape.global_units(list(range(scn.R))).reshape(-1).numpy()
    out = {}
    for u in range(scn.U):
        recs = []
        for cls, n in ((1, o.n_h[u]), (2, o.n_l[u])):
            for s in range(int(n)):
                kc, km, vc, vm, sg, ps = o.slot_record(cls, u, s)
                recs.append((ps, cls, sg, km, vm, kc.tobytes(), vc.tobytes()))
        out[int(ug[u])] = tuple(sorted(recs))
    return out


def _run(scn, steps):
    o = H.OracleBackend(scn)
    inp = H.Inputs(scn)
    life = H.Lifecycle(scn)
    H.admit([o], inp, life, list(range(scn.R)), [40] * scn.R)
    for step in range(steps):
        H.decode_step([o], inp, life, step)
    return o


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        base = H.TINY.replace(R=2, Ly=2, H=4, d=32, W=8, Ch=4, Cl=8, M=96, P=600, seed=21)
        h0, hl = shard_heads(base.H, world, rank)
        scn = base.replace(H=hl, H_total=base.H, h0=h0)
        o = _run(scn, steps=12)
        mine = _unit_contents(o, scn)
        # count all-reduce over the two pools
        stats = torch.tensor([o.pool.free, -o.pool.last_demand, -(scn.P - o.pool.free), o.pool.status],
                             dtype=torch.int64)
        red, _ = count_allreduce(stats)
        gathered = [None] * world
        dist.all_gather_object(gathered, (mine, stats.tolist(), red.tolist()))
        if rank == 0:
            full = _unit_contents(_run(base, steps=12), base)
            merged = {}
            for m, _, _ in gathered:
                merged.update(m)
            q.put(dict(same=merged == full, n=len(full),
                       stats=[g[1] for g in gathered], red=gathered[0][2], red1=gathered[1][2]))
    finally:
        dist.destroy_process_group()


def test_head_sharded_pools_match_single_pool_and_count_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, q), nprocs=2, join=True)
    res = q.get()
    assert res["n"] == 2 * 2 * 4
    assert res["same"], "sharded pools differ from the single pool (PIN-13)"
    s0, s1 = res["stats"]
    assert res["red"] == res["red1"] == [min(a, b) for a, b in zip(s0, s1)]


def _error_worker(rank, world, port, q):
    """rank 1's pool runs out of pages at admission (a real sticky OOM); rank 0's is healthy"""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scn = H.TINY.replace(R=2, Ly=2, H=2, d=32, W=8, Ch=4, Cl=8, M=96, P=600 if rank == 0 else 20, seed=5)
        o = H.OracleBackend(scn)
        inp = H.Inputs(scn)
        sig, k, v = inp.prefill([0, 1], [60, 60])
        assert o.classify_prefill([0, 1], [60, 60], sig) == 0
        o.compact_alloc(None)
        p = o.pool
        stats = torch.tensor([p.free, -p.last_demand, -(scn.P - p.free), p.status], dtype=torch.int64)
        red, _ = count_allreduce(stats)
        adm = Admission(decode_reserve=0)
        q.put((rank, int(p.status), red.tolist(), adm.healthy(red), adm.admit(red, 0)))
    finally:
        dist.destroy_process_group()


def test_count_allreduce_shows_an_error_on_one_rank():
    """the counters carry status itself (<= 0), so the MIN is negative when any one GPU has a pending
    error and admission stops on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.spawn(_error_worker, args=(2, _free_port(), q), nprocs=2, join=True)
    res = sorted([q.get(), q.get()])
    assert res[0][1] == 0 and res[1][1] == -3                            # rank 1: DKV_ERR_OOM
    for _, _, red, healthy, admit in res:
        assert red[3] == -3 and not healthy and not admit


def test_shard_heads_and_admission_rule():
    assert [shard_heads(8, 4, r) for r in range(4)] == [(0, 2), (2, 2), (4, 2), (6, 2)]
    with pytest.raises(ValueError):
        shard_heads(8, 3, 0)
    adm = Admission(decode_reserve=100)
    b = prefill_page_bound(4096, 64, 16, units=256)
    assert b == 256 * (252 + 1)
    assert adm.admit(torch.tensor([b + 100, -5, -10, 0]), b)
    assert not adm.admit(torch.tensor([b + 99, -5, -10, 0]), b)
    assert not adm.admit(torch.tensor([b + 1000, -5, -10, -3]), b)      # a GPU reports OOM
