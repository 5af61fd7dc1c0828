"""GPU-vs-oracle parity through the C ABI: bit-exact decisions, ring, pointers, tables, counts, request
state, window and page bytes after EVERY call, on seeded synthetic lifecycles (prefill, decode with
significance drift, frees, re-admission)."""
import numpy as np
import pytest
import torch

from tests import harness as H

pytestmark = pytest.mark.gpu


def _mk(scn):
    from tests.gpu_backend import GpuBackend
    return H.OracleBackend(scn), GpuBackend(scn)


def _lifecycle(scn, steps, prompt_lens, frees=(), readmit_len=None, pages_every=1, tol_steps=None, head=None):
    from tests.gpu_backend import compare_state, dec_np
    o, g = _mk(scn)
    if head is not None:                                         # NEXT-4: per-head thresholds on both sides
        assert o.set_head_thresholds(*head) == 0 and g.set_head_thresholds(*head) == 0
    inp = H.Inputs(scn)
    life = H.Lifecycle(scn)
    counter = {"n": 0}

    def check(where, decs=None):
        counter["n"] += 1
        if decs is not None:
            a, b = dec_np(decs[0]), dec_np(decs[1])
            if not np.array_equal(a.view(np.uint8), b.view(np.uint8)):
                bad = np.nonzero(a != b)[0]
                raise AssertionError(f"[{where}] decisions differ at units {bad[:8].tolist()}: oracle {a[bad[0]]} gpu {b[bad[0]]}")
        with_pages = (counter["n"] % pages_every == 0) or where.endswith("prefill")
        so, sg = o.snapshot(pages=with_pages), g.snapshot(pages=with_pages)
        compare_state(so, sg, where=where)
        assert sg["status"] == 0, f"[{where}] device status {sg['status']}"

    reqs = list(range(len(prompt_lens)))
    H.admit([o, g], inp, life, reqs, prompt_lens, check=check)
    pending = {}
    frees = dict(frees)
    for step in range(steps):
        H.decode_step([o, g], inp, life, step, check=check)
        for r, t in list(pending.items()):
            if step >= t and o.pool.req_state[r] == 0:
                H.admit([o, g], inp, life, [r], [readmit_len or prompt_lens[r]], check=check)
                del pending[r]
        if step in frees:
            H.free([o, g], life, frees[step])
            check(f"free@{step}")
            for r in frees[step]:
                pending[r] = step + 1
    return o, g, life


def test_tiny_parity_every_call():
    # BASELINE configs[0]: 4 requests x 2 layers x 4 KV heads, head_dim 64, 64-token prompts, 16-token pages,
    # 1024 pages; 64 decode steps, one request freed at step 32 and re-admitted
    _lifecycle(H.TINY, steps=64, prompt_lens=[64, 64, 64, 64], frees=[(32, [1])], readmit_len=48)


@pytest.mark.parametrize("tile_units", [256, 1024])
def test_multi_tile_ragged_parity(tile_units):
    # U = 7 * 5 * 40 = 1400 units: 6 tiles of 256 (ragged tail 120) or 2 of 1024; d = 128, K8V4/K4V2,
    # W = 64, ragged prompt lengths (some <= W), frees of several requests in one step
    scn = H.TINY.replace(R=7, Ly=5, H=40, d=128, M=1100, W=64, P=40000, seed=11, tile_units=tile_units)
    lens = [300, 64, 517, 40, 0, 1000, 129]
    _lifecycle(scn, steps=40, prompt_lens=lens, frees=[(12, [0, 2]), (25, [5])], readmit_len=260, pages_every=7)


def test_prompt_denominator_and_qwen_thresholds_parity():
    # Q4's alternative reading (alpha / n) and the Qwen/QwQ thresholds alpha_h = 3, alpha_l = 0 (Q24)
    scn = H.TINY.replace(R=3, Ly=3, H=8, d=128, M=512, W=32, P=6000, alpha_h=3.0, alpha_l=0.0,
                         prompt_denominator=1, seed=5, mix=(0.40, 0.60, 0.0))
    _lifecycle(scn, steps=30, prompt_lens=[200, 333, 90], frees=[(10, [1])], readmit_len=120)


def test_tile_size_determinism():
    # PIN-14: the decoupled look-back order must not leak into results
    scn = H.TINY.replace(R=6, Ly=4, H=50, d=64, M=300, W=16, P=30000, seed=3)
    from tests.gpu_backend import GpuBackend
    snaps = []
    for tu in (256, 512, 1024):
        g = GpuBackend(scn.replace(tile_units=tu))
        inp = H.Inputs(scn)
        life = H.Lifecycle(scn)
        H.admit([g], inp, life, list(range(6)), [200, 17, 256, 100, 5, 150])
        for step in range(20):
            H.decode_step([g], inp, life, step)
            if step == 7:
                H.free([g], life, [2, 3])
        snaps.append(g.snapshot())
    from tests.gpu_backend import compare_state
    compare_state(snaps[0], snaps[1], where="256 vs 512")
    compare_state(snaps[0], snaps[2], where="256 vs 1024")


# ---------------------------------------------------------------- NEXT-1: the paper's prompt workflow
@pytest.mark.parametrize("tile_units", [256, 1024])
def test_prompt_workflow_parity(tile_units):
    # prefill_workflow = 1: conservative blocks, top-ups (Q29), reclaimed middles — ring,
    # pointers, tables, counts and page bytes bit-exact with the oracle after every call, across several
    # scan tiles with a ragged tail, frees and re-admission
    scn = H.TINY.replace(R=7, Ly=5, H=40, d=128, M=1100, W=64, P=60000, seed=23, tile_units=tile_units,
                         prefill_workflow=1)
    lens = [300, 64, 517, 40, 0, 1000, 129]
    _lifecycle(scn, steps=24, prompt_lens=lens, frees=[(7, [0, 2]), (15, [5])], readmit_len=260, pages_every=5)


def test_prompt_workflow_tiny_and_wraparound():
    # the free region ends at the allocation pointer (fresh pool): reclaimed middles wrap onto granted ring
    # slots, which the kernel must read before the reclaim writes land (second grid barrier)
    scn = H.TINY.replace(prefill_workflow=1, P=700)
    _lifecycle(scn, steps=40, prompt_lens=[64, 64, 64, 64], frees=[(20, [1, 3])], readmit_len=48)


def test_fig5_on_gpu():
    """PIN-1 at GPU level: Fig. 5 with every token doubled (4-token high / 8-token low pages;
    the CUDA geometry needs C % 4 == 0) — pages 5-8 -> head A, 9-12 -> head B, A keeps 5 + 8, B keeps
    9, 10 + 12, pages 6, 7, 11 reclaimed at the end pointer, which wraps to the head of the list."""
    import json
    import os
    from paper_2412_03131_b200 import Pool
    from paper_2412_03131_b200 import dkv as D
    with open(os.path.join(os.path.dirname(__file__), "golden", "fig5.json")) as f:
        g = json.load(f)
    cfg = D.make_config(R=1, Ly=1, H=2, d=64, M=16, W=0, Ch=4, Cl=8, P=16, alpha_h=1.0, alpha_l=0.02,
                        prefill_workflow=1)
    pool = Pool(cfg, device="cuda")
    v = pool.views()
    v["ctrl"][0] = g["initial"]["start"]                  # pages 0-4 held outside the example (as in Fig. 5)
    v["ctrl"][1] = g["initial"]["free"]
    torch.cuda.synchronize()
    n0 = g["prompt_len"]
    sig = np.repeat(np.array(g["sig"], np.float32), 2, axis=1)
    i = np.arange(1, 2 * n0 + 1, dtype=np.float32)
    base = np.repeat(np.arange(1, n0 + 1, dtype=np.float32), 2)
    sig = (sig * (base / i)).astype(np.float32).reshape(1, 2, 2 * n0)   # each token keeps its Fig. 5 class
    pool.classify_prefill([0], [2 * n0], torch.from_numpy(sig).cuda())
    pool.compact_alloc(None)
    st, stats = pool.query()
    assert st == 0
    e = g["expect"]
    table = v["table"].cpu().numpy()
    L = table.shape[1]
    for head, u in (("A", 0), ("B", 1)):
        assert list(table[u, :len(e["high_pages"][head])]) == e["high_pages"][head]
        assert [int(table[u, L - 1 - k]) for k in range(len(e["low_pages"][head]))] == e["low_pages"][head]
    ring = v["ring"].cpu().numpy()
    assert list(ring[:3]) == e["ring_head_after"]
    ctrl = v["ctrl"].cpu().numpy()
    assert int(ctrl[0]) == e["start_after"] and int(ctrl[1]) == e["free_after"]
    free_region = [int(ring[(int(ctrl[0]) + k) % 16]) for k in range(int(ctrl[1]))]
    assert free_region == e["free_region_after"]


# ---------------------------------------------------------------- NEXT-4: per-head thresholds (Q35)
@pytest.mark.parametrize("workflow", [0, 1])
def test_per_head_thresholds_parity(workflow):
    scn = H.TINY.replace(R=5, Ly=3, H=6, d=128, M=700, W=32, P=30000, seed=41, tile_units=256,
                         prefill_workflow=workflow)
    rng = np.random.default_rng(41)
    n = scn.Ly * scn.H
    ah = rng.choice([0.5, 1.0, 3.0, 1e30], size=n).astype(np.float32)
    al = rng.choice([0.0, 0.02, 0.1, 1e30], size=n).astype(np.float32)
    _lifecycle(scn, steps=20, prompt_lens=[300, 64, 200, 17, 450], frees=[(8, [1, 3])], readmit_len=150,
               pages_every=4, head=(ah, al))


@pytest.mark.parametrize("path", ["fast", "barrier"])
def test_many_tiles_lookback_window_parity(path):
    """the decoupled look-back slides its 32-predecessor window (`look -= 32`) only when more
    than 33 tiles precede a tile.  U = 12 x 32 x 32 = 12288 units at 256-unit tiles = 48 tiles; the whole ring,
    both pointers, every table and count compared with the oracle after every call.  "fast": free >= U, the
    decode scan has no grid barrier; "barrier": a pool tight enough that free < U, so every decode call takes
    the all-or-nothing barrier path (prefill always does).  Frees of several requests in one step."""
    base = H.TINY.replace(R=12, Ly=32, H=32, d=64, M=160, W=16, seed=41, tile_units=256)
    assert base.U // 256 >= 34
    lens = [40, 24, 56, 33, 17, 48, 60, 29, 44, 36, 52, 20]
    if path == "fast":
        scn = base.replace(P=200000)
    else:
        probe = H.OracleBackend(base.replace(P=200000))
        inp, life = H.Inputs(base), H.Lifecycle(base)
        H.admit([probe], inp, life, list(range(12)), lens)
        used = 200000 - probe.pool.free
        scn = base.replace(P=used + base.U // 2)               # free < U from the first decode step
    o, g, life = _lifecycle(scn, steps=12, prompt_lens=lens, frees=[(3, [2, 7]), (6, [0, 5, 11])],
                            readmit_len=30, pages_every=5)
    if path == "barrier":
        assert o.pool.free < scn.U
