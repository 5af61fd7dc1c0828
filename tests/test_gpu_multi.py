"""The N-rank path on CUDA pools (rows a9 / e: "each worker includes a dedicated memory manager that
oversees the KV cache for its assigned attention heads").  Two processes share cuda:0 (the GPU box has one
GPU), each holding an independent CUDA pool for its half of the KV heads; the per-step count all-reduce runs
over gloo (NCCL refuses two ranks on one device — on an 8-GPU node bench.py uses NCCL, one GPU per rank).
Every rank's pool is bit-exact with an oracle pool of the same shard after every call, and the reduced
counters equal the element-wise MIN of both ranks' counters, which equal the oracle's.  A second test runs
`bench.py --gpus 2 --shared-device` and checks that its line reports two ranks."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import harness as H

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_03131_b200.admission import count_allreduce, shard_heads
        from tests.gpu_backend import GpuBackend, compare_state, dec_np
        torch.cuda.set_device(0)
        base = H.TINY.replace(R=6, Ly=3, H=4, d=64, W=16, M=200, P=4000, seed=31, tile_units=256)
        h0, hl = shard_heads(base.H, world, rank)
        scn = base.replace(H=hl, H_total=base.H, h0=h0)
        o, g = H.OracleBackend(scn), GpuBackend(scn, device="cuda:0")
        inp, life = H.Inputs(scn), H.Lifecycle(scn)
        n_checked = 0

        def check(where, decs=None):
            nonlocal n_checked
            if decs is not None:
                assert np.array_equal(dec_np(decs[0]).view(np.uint8), dec_np(decs[1]).view(np.uint8)), where
            compare_state(o.snapshot(), g.snapshot(), where=f"rank {rank} {where}")
            n_checked += 1

        H.admit([o, g], inp, life, list(range(scn.R)), [40 + 9 * r for r in range(scn.R)], check=check)
        reduced = []
        for step in range(20):
            H.decode_step([o, g], inp, life, step, check=check)
            if step == 6:
                H.free([o, g], life, [1, 4])
            if step == 9:
                H.admit([o, g], inp, life, [1], [77], check=check)
            torch.cuda.synchronize()
            st_gpu = g.pool.views()["stats"].cpu().clone()
            p = o.pool
            st_orc = torch.tensor([p.free, -p.last_demand, -(scn.P - p.free), p.status], dtype=torch.int64)
            assert torch.equal(st_gpu, st_orc), (rank, step, st_gpu.tolist(), st_orc.tolist())
            red, _ = count_allreduce(st_gpu)
            gathered = [None] * world
            dist.all_gather_object(gathered, st_gpu.tolist())
            assert red.tolist() == [min(a, b) for a, b in zip(*gathered)], (rank, step)
            reduced.append(red.tolist())
        q.put((rank, n_checked, reduced))
    finally:
        dist.destroy_process_group()


def test_two_rank_cuda_pools_match_oracle_shards_and_min_counters():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.spawn(_worker, args=(2, _free_port(), q), nprocs=2, join=True)
    res = sorted([q.get(), q.get()])
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] > 60 for r in res)                     # every call of every step compared
    assert res[0][2] == res[1][2]                          # both ranks see the same reduced counters


def test_bench_two_ranks_report_two_gpus():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "tiny", "--gpus", "2",
                          "--shared-device", "--steps", "3", "--warmup", "3", "--next2", "0"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["dist"]["world"] == 2 and line["dist"]["backend"] == "gloo"
    assert line["quant_write"]["gbs"] > 0 and line["value"] > 0


def test_bench_refuses_more_ranks_than_gpus():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    n = torch.cuda.device_count() + 1
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "tiny", "--gpus", str(n),
                          "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env,
                         cwd=ROOT)
    assert out.returncode != 0 and "CUDA device" in out.stderr
