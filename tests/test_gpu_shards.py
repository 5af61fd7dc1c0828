"""PIN-13 on the CUDA path: the same global workload run as one pool holding all KV heads and as N pools each
holding a head shard (one pool per GPU at N GPUs; here all on one device) stores identical logical
content for every global unit — classes, codes, metadata, scores, positions — at N = 1, 2, 4, 8; page IDs
differ by design.  Also checks each shard against the oracle shard bit for bit."""
import numpy as np
import pytest
import torch

from tests import harness as H

pytestmark = pytest.mark.gpu


def _contents(g, scn):
    """global unit -> sorted per-slot records from a GPU pool (device views, page IDs excluded)"""
    v = g.pool.views()
    pages, table = v["pages"].cpu().numpy(), v["table"].cpu().numpy()
    n_h, n_l = v["n_h"].cpu().numpy(), v["n_l"].cpu().numpy()
    geom, L = g.geom, g.L
    ug = scn.shape.global_units(list(range(scn.R))).reshape(-1).numpy()
    out = {}
    for u in range(scn.U):
        recs = []
        for cls, n in ((1, n_h[u]), (2, n_l[u])):
            gg = geom[cls]
            for s in range(int(n)):
                pid = table[u, s // gg["C"]] if cls == 1 else table[u, L - 1 - s // gg["C"]]
                i = s % gg["C"]
                pg = pages[pid]
                recs.append((int(pg[gg["off_pos"] + 4 * i: gg["off_pos"] + 4 * i + 4].view(np.int32)[0]), cls,
                             pg[gg["off_score"] + 4 * i: gg["off_score"] + 4 * i + 4].tobytes(),
                             pg[gg["off_kmeta"] + 4 * i: gg["off_kmeta"] + 4 * i + 4].tobytes(),
                             pg[gg["off_vmeta"] + 4 * i: gg["off_vmeta"] + 4 * i + 4].tobytes(),
                             pg[gg["off_k"] + i * gg["k_row"]: gg["off_k"] + (i + 1) * gg["k_row"]].tobytes(),
                             pg[gg["off_v"] + i * gg["v_row"]: gg["off_v"] + (i + 1) * gg["v_row"]].tobytes()))
        out[int(ug[u])] = tuple(sorted(recs))
    return out


def _run_shard(scn, steps, with_oracle):
    from tests.gpu_backend import GpuBackend, compare_state
    g = GpuBackend(scn)
    backends = [g]
    o = None
    if with_oracle:
        o = H.OracleBackend(scn)
        backends = [o, g]
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit(backends, inp, life, list(range(scn.R)), [150, 90, 200][: scn.R])
    for step in range(steps):
        H.decode_step(backends, inp, life, step)
        if step == 6:
            H.free(backends, life, [1])
    if o is not None:
        compare_state(o.snapshot(), g.snapshot(), where=f"shard h0={scn.h0}")
    return g


def test_head_shards_store_the_same_content():
    base = H.TINY.replace(R=3, Ly=2, H=8, d=128, M=400, W=32, P=20000, seed=17)
    full = _contents(_run_shard(base, 14, with_oracle=False), base)
    for n in (2, 4, 8):
        merged = {}
        hl = base.H // n
        for rank in range(n):
            scn = base.replace(H=hl, H_total=base.H, h0=rank * hl)
            merged.update(_contents(_run_shard(scn, 14, with_oracle=(n == 4)), scn))
        assert merged == full, f"sharded {n}-way differs from the single pool"
