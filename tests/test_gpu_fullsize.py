"""Parity at BASELINE.json's full size (configs[1]: 64 requests x 32 layers x 8 KV heads, head_dim 128,
4096-token prompts, 2^22 pages) in the launch configuration bench.py times, on sampled requests the
oracle recomputes one by one (a sub-pool holding only those requests: their units see the same inputs,
and every unit's slot contents depend only on its own history), plus pool-wide properties that hold at any
size (page ownership is a permutation, occupied slots are exactly [0, ph) u [L - pl, L))."""
import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _unit_records(pages, table_row, n_h, n_l, geom, L):
    """per-slot (k codes, k meta, v codes, v meta, score bits, pos) of one unit from device tensors"""
    recs = {}
    for cls, n in ((1, n_h), (2, n_l)):
        g = geom[cls]
        C = g["C"]
        npg = -(-int(n) // C)
        if npg == 0:
            continue
        cols = list(range(npg)) if cls == 1 else [L - 1 - k for k in range(npg)]
        pids = table_row[cols].long()
        pg = pages[pids].cpu().numpy()                                  # [npg, page_bytes]
        for s in range(int(n)):
            b = pg[s // C]
            i = s % C
            recs[(cls, s)] = (b[g["off_k"] + i * g["k_row"]: g["off_k"] + (i + 1) * g["k_row"]].tobytes(),
                              b[g["off_kmeta"] + 4 * i: g["off_kmeta"] + 4 * i + 4].tobytes(),
                              b[g["off_v"] + i * g["v_row"]: g["off_v"] + (i + 1) * g["v_row"]].tobytes(),
                              b[g["off_vmeta"] + 4 * i: g["off_vmeta"] + 4 * i + 4].tobytes(),
                              b[g["off_score"] + 4 * i: g["off_score"] + 4 * i + 4].tobytes(),
                              b[g["off_pos"] + 4 * i: g["off_pos"] + 4 * i + 4].tobytes())
    return recs


def _section(pages, table_row, n, C, off_score, off_pos, cls, L):
    """score bits (u32) and positions of a section's n slots in slot order, from a device tensor or a host array"""
    npg = -(-n // C)
    cols = np.arange(npg) if cls == 1 else L - 1 - np.arange(npg)
    pids = np.asarray(table_row)[cols].astype(np.int64)
    if isinstance(pages, torch.Tensor):
        pg = pages[torch.from_numpy(pids).to(pages.device)].cpu().numpy()
    else:
        pg = pages[pids]
    sc = np.ascontiguousarray(pg[:, off_score:off_score + 4 * C]).view(np.uint32).reshape(-1)[:n]
    ps = np.ascontiguousarray(pg[:, off_pos:off_pos + 4 * C]).view(np.int32).reshape(-1)[:n]
    return sc, ps


def test_llama8b_fullsize_sampled_parity():
    import bench
    import synth
    from paper_2412_03131_b200 import Pool, decisions_to_numpy
    from paper_2412_03131_b200 import dkv as D
    from tests import harness as H

    c = bench.CONFIGS["llama3_8b"]
    dev = torch.device("cuda", 0)
    wl = bench.Workload(c, 0, 1, dev)
    T = c["prompt"]
    cfg = D.make_config(wl.R, c["Ly"], wl.Hl, c["d"], c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"],
                        alpha_h=c["alpha_h"], alpha_l=c["alpha_l"])
    pool = Pool(cfg, device=dev)
    geom, L, LyH = pool.geom(), pool.L, pool.LyH
    sig, kk, vv = wl.prefill_inputs(T)
    reqs = list(range(wl.R))
    pool.classify_prefill(reqs, [T] * wl.R, sig)
    pool.compact_alloc(None)
    pool.quant_write_prefill(kk.view(torch.int16), vv.view(torch.int16), sig)
    del kk, vv
    dec = pool.new_decisions()

    sample = (0, 37)
    scn = H.Scenario(R=2, Ly=c["Ly"], H=c["H"], d=c["d"], M=c["M"], W=c["W"], Ch=c["Ch"], Cl=c["Cl"],
                     P=2 * LyH * (T // c["Ch"] + 8), alpha_h=c["alpha_h"], alpha_l=c["alpha_l"], seed=c["seed"],
                     mix=c["mix"], req_ids=sample)
    o = H.OracleBackend(scn)
    inp = H.Inputs(scn)                                                  # oracle inputs drawn on the host
    life = H.Lifecycle(scn)
    H.admit([o], inp, life, [0, 1], [T, T])

    def compare(where, dec_gpu=None, dec_orc=None):
        torch.cuda.synchronize()
        v = pool.views()
        n_h, n_l = v["n_h"].cpu().numpy(), v["n_l"].cpu().numpy()
        for i, r in enumerate(sample):
            for j in range(LyH):
                ug, uo = r * LyH + j, i * LyH + j
                assert (n_h[ug], n_l[ug]) == (o.pool.n_h[uo], o.pool.n_l[uo]), (where, r, j)
                if j % 37 == 0 or dec_gpu is not None:
                    a = _unit_records(v["pages"], v["table"][ug], n_h[ug], n_l[ug], geom, L)
                    b = {}
                    for cls, n in ((1, o.pool.n_h[uo]), (2, o.pool.n_l[uo])):
                        for s in range(int(n)):
                            kc, km, vc, vm, sg, ps = o.pool.slot_record(cls, uo, s)
                            b[(cls, s)] = (kc.tobytes(), np.uint32(km).tobytes(), vc.tobytes(),
                                           np.uint32(vm).tobytes(), np.uint32(sg).tobytes(), np.int32(ps).tobytes())
                    assert a == b, (where, r, j)
                    wk = v["win_k"][ug].cpu().numpy().view(np.uint16)
                    assert np.array_equal(wk, o.pool.win_k[uo]), (where, r, j)
            if dec_gpu is not None:
                a = dec_gpu[r * LyH:(r + 1) * LyH]
                b = dec_orc[i * LyH:(i + 1) * LyH]
                assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (where, r)
        # pool-wide properties at full size (on the device)
        ctrl = v["ctrl"].cpu().numpy()
        start, free, P = int(ctrl[0]), int(ctrl[1]), c["P"]
        ring = v["ring"]
        free_ids = ring[(start + torch.arange(free, device=dev)) % P]
        tab = v["table"]
        used = tab[tab >= 0]
        allids = torch.cat([free_ids, used]).sort().values
        assert allids.numel() == P and torch.equal(allids, torch.arange(P, device=dev, dtype=allids.dtype)), where
        ph = (v["n_h"].long() + c["Ch"] - 1) // c["Ch"]
        pl = (v["n_l"].long() + c["Cl"] - 1) // c["Cl"]
        k = torch.arange(L, device=dev).view(1, -1)
        expect = (k < ph.view(-1, 1)) | (k >= (L - pl).view(-1, 1))
        assert torch.equal(tab >= 0, expect), where

    compare("prefill")
    seq = np.full(wl.R, T, np.int64)
    act = np.ones(wl.R, bool)
    for step in range(3):
        v = pool.views()
        synth.apply_drift(c["seed"], step, wl.shape, v["pages"], v["table"], v["n_h"], v["n_l"],
                          {k_: (geom[k_]["C"], geom[k_]["off_score"], geom[k_]["off_pos"]) for k_ in (1, 2)}, L)
        cand, nk, nv = wl.decode_inputs(seq, act)
        pool.classify_decode(cand, dec)
        pool.compact_alloc(dec)
        pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), cand)
        seq += 1
        decs = H.decode_step([o], inp, life, step)
        compare(f"decode {step}", decisions_to_numpy(dec), decs[0])
    st, _ = pool.query()
    assert st == 0


def test_synth_generators_device_independent():
    """The input generators give bit-identical values on the host and on the device (so the bench may draw
    its 32 GiB of inputs on the GPU while the oracle draws its sample on the host)."""
    import synth
    ug = torch.arange(0, 4096, 7, dtype=torch.int64)
    a =synth.kv_values(5, synth.S_KEY, ug, 0, 64, 128)
    b = synth.kv_values(5, synth.S_KEY, ug.cuda(), 0, 64, 128).cpu()
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    mh, ml = synth.unit_mix(5, ug, Ly=32, Ht=8)
    s1 = synth.prefill_sig(5, ug, 300, 1.0, 0.02, mh, ml)
    s2 = synth.prefill_sig(5, ug.cuda(), 300, 1.0, 0.02, mh.cuda(), ml.cuda()).cpu()
    assert torch.equal(s1.view(torch.int32), s2.view(torch.int32))
    N = torch.full((ug.numel(),), 4500, dtype=torch.int64)
    d1 = synth.decode_sig(5, ug, N, 64, 1.0, 0.02, mh, ml)
    d2 = synth.decode_sig(5, ug.cuda(), N.cuda(), 64, 1.0, 0.02, mh.cuda(), ml.cuda()).cpu()
    assert torch.equal(d1.view(torch.int32), d2.view(torch.int32))


def test_llama8b_fullsize_attention_sampled_parity():
    """NEXT-2 at the bench's full size and launch configuration (configs[1], q_per_kv 4 as bench.py times it):
    dkv_attend over all 16384 units, then a decode step whose classify takes t_c's significance from the window
    and its victims from the attention kernel's section minima (d_sig NULL).  Two sampled requests (512 units)
    are recomputed by the oracle one by one: attention outputs, the significance written back (every stored
    slot's score bits, the window significance), the section minima and the following decisions are bit-exact."""
    import bench
    from paper_2412_03131_b200 import Pool, decisions_to_numpy
    from paper_2412_03131_b200 import dkv as D
    from tests import harness as H
    from tests.gpu_backend import dec_np

    c = bench.CONFIGS["llama3_8b"]
    G, d = c["G"], c["d"]
    dev = torch.device("cuda", 0)
    wl = bench.Workload(c, 0, 1, dev)
    T = c["prompt"]
    cfg = D.make_config(wl.R, c["Ly"], wl.Hl, d, c["M"], c["W"], c["Ch"], c["Cl"], P=c["P"],
                        alpha_h=c["alpha_h"], alpha_l=c["alpha_l"], q_per_kv=G)
    pool = Pool(cfg, device=dev)
    geom, L, LyH = pool.geom(), pool.L, pool.LyH
    sig, kk, vv = wl.prefill_inputs(T)
    reqs = list(range(wl.R))
    pool.classify_prefill(reqs, [T] * wl.R, sig)
    pool.compact_alloc(None)
    pool.quant_write_prefill(kk.view(torch.int16), vv.view(torch.int16), sig)
    del kk, vv, sig

    sample = (5, 62)
    scn = H.Scenario(R=2, Ly=c["Ly"], H=c["H"], d=d, M=c["M"], W=c["W"], Ch=c["Ch"], Cl=c["Cl"],
                     P=2 * LyH * (T // c["Ch"] + 8), alpha_h=c["alpha_h"], alpha_l=c["alpha_l"], seed=c["seed"],
                     mix=c["mix"], req_ids=sample, q_per_kv=G)
    o = H.OracleBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o], inp, life, [0, 1], [T, T])
    rows = np.concatenate([np.arange(r * LyH, (r + 1) * LyH) for r in sample])
    rng = np.random.default_rng(11)

    def attend_and_compare(where):
        q = rng.normal(0, 1, size=(wl.U, G, d)).astype(np.float16)
        out = torch.empty((wl.U, G, d), dtype=torch.float32, device=dev)
        assert pool.attend(torch.from_numpy(q.view(np.int16)).to(dev), out) == 0
        st, oo, _ = o.attend(q[rows], want_out=True, want_probs=False)
        assert st == 0
        og = out.cpu().numpy()[rows]
        assert np.array_equal(oo.view(np.uint32), og.view(np.uint32)), f"[{where}] attention outputs differ"
        v = pool.views()
        # the GPU outputs of 64 sampled units pinned to Eq. 1 evaluated in float64 from the GPU's page bytes
        from tests import eq1
        snap = dict(pages=v["pages"], table=v["table"], n_h=v["n_h"], n_l=v["n_l"], seq_len=v["seq_len"],
                    win_k=v["win_k"], win_v=v["win_v"])
        out_np = out.cpu().numpy()
        eq1.check_units(snap, geom, L, c["W"], d, LyH, q, out_np, None, range(0, wl.U, wl.U // 64), where=where)
        n_h, n_l = v["n_h"].cpu().numpy(), v["n_l"].cpu().numpy()
        secmin = v["secmin"].cpu().numpy()
        win_sig = v["win_sig"].cpu().numpy()
        gtab = v["table"][torch.from_numpy(rows).to(dev)].cpu().numpy()
        for i, r in enumerate(sample):
            for j in range(LyH):
                ug, uo = r * LyH + j, i * LyH + j
                assert (n_h[ug], n_l[ug]) == (o.pool.n_h[uo], o.pool.n_l[uo]), (where, r, j)
                for k, cls in enumerate((1, 2)):
                    n = int(o.pool.n_h[uo] if cls == 1 else o.pool.n_l[uo])
                    if n == 0:
                        continue
                    # every stored slot's significance (score bits) and position after the write-back
                    gs, gp = _section(v["pages"], gtab[i * LyH + j], n, geom[cls]["C"], geom[cls]["off_score"],
                                      geom[cls]["off_pos"], cls, L)
                    og_ = o.pool.geom[cls]
                    os_, op_ = _section(o.pool.pages, o.pool.table[uo], n, og_.C, og_.off_score, og_.off_pos, cls, L)
                    assert np.array_equal(gs, os_) and np.array_equal(gp, op_), (where, r, j, cls)
                    # the section minimum the next classify uses: (significance bits, position, slot)
                    key = (os_.astype(np.uint64) << np.uint64(32)) | op_.astype(np.uint32).astype(np.uint64)
                    s_min = int(np.argmin(key))
                    want = (int(os_[s_min].view(np.int32)), int(op_[s_min]), s_min)
                    assert tuple(int(x) for x in secmin[ug][3 * k:3 * k + 3]) == want, (where, r, j, cls)
                assert np.array_equal(win_sig[ug].view(np.uint32), o.pool.win_sig[uo].view(np.uint32)), (where, r, j)

    attend_and_compare("prefill")
    dec = pool.new_decisions()
    seq = np.full(wl.R, T, np.int64)
    act = np.ones(wl.R, bool)
    for step in range(2):
        _, nk, nv = wl.decode_inputs(seq, act)
        pool.classify_decode(None, dec)
        pool.compact_alloc(dec)
        pool.quant_write_decode(dec, nk.view(torch.int16), nv.view(torch.int16), None)
        seq += 1
        active = life.state == H.REQ_ACTIVE
        N = np.where(active, life.seq + 1, 0)
        _, k, v_ = inp.decode(N)
        st, do = o.classify_decode(None)
        assert st == 0
        assert o.compact_alloc(do) == 0 and o.quant_write_decode(do, k, v_, None) == 0
        life.seq[active] += 1
        dg, dor = dec_np(decisions_to_numpy(dec)), dec_np(do)
        for i, r in enumerate(sample):
            a = np.ascontiguousarray(dg[r * LyH:(r + 1) * LyH])
            b = np.ascontiguousarray(dor[i * LyH:(i + 1) * LyH])
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), (step, r)
        attend_and_compare(f"decode {step}")
    st, _ = pool.query()
    assert st == 0


def test_llama8b_fullsize_attention_tc_sampled_and_deterministic():
    """NEXT-2 on tensor cores at the bench's full size and launch configuration (configs[1], q_per_kv 4, 16384
    units over the persistent CTAs, each CTA's significance pass deferred into its next unit): outputs and per-token
    scores of 64 sampled units against Eq. 1 in float64 from the pool's page bytes; the significance written back
    for those units against the float64 running mean (Q33); and the whole call deterministic — re-run from the same
    arena bytes it produces bit-identical outputs, scores and arena (a race check in the absence of the sanitizer)."""
    import bench
    from paper_2412_03131_b200 import Pool
    from paper_2412_03131_b200 import dkv as D
    from tests import eq1

    c = bench.CONFIGS["llama3_8b"]
    G, d, W = c["G"], c["d"], c["W"]
    dev = torch.device("cuda", 0)
    wl = bench.Workload(c, 0, 1, dev)
    T = c["prompt"]
    cfg = D.make_config(wl.R, c["Ly"], wl.Hl, d, c["M"], W, c["Ch"], c["Cl"], P=c["P"],
                        alpha_h=c["alpha_h"], alpha_l=c["alpha_l"], q_per_kv=G)
    pool = Pool(cfg, device=dev)
    geom, L, LyH = pool.geom(), pool.L, pool.LyH
    sig, kk, vv = wl.prefill_inputs(T)
    pool.classify_prefill(list(range(wl.R)), [T] * wl.R, sig)
    pool.compact_alloc(None)
    pool.quant_write_prefill(kk.view(torch.int16), vv.view(torch.int16), sig)
    del kk, vv, sig
    q = np.random.default_rng(3).normal(0, 1, size=(wl.U, G, d)).astype(np.float16)
    qd = torch.from_numpy(q.view(np.int16)).to(dev)
    sample = list(range(0, wl.U, wl.U // 64))
    v = pool.views()
    torch.cuda.synchronize()
    before = {u: _unit_scores(v, geom, L, u) for u in sample}
    arena0 = pool.arena.clone()
    runs = []
    for rep in range(2):
        if rep:
            pool.arena.copy_(arena0)
        out = torch.empty((wl.U, G, d), dtype=torch.float32, device=dev)
        probs = torch.zeros((wl.U, c["M"]), dtype=torch.float32, device=dev)
        assert pool.attend_tc(qd, out, probs) == 0
        torch.cuda.synchronize()
        runs.append((out, probs, pool.arena.clone() if rep == 0 else None))
    assert torch.equal(runs[0][0], runs[1][0]) and torch.equal(runs[0][1], runs[1][1]), "attend_tc not deterministic"
    assert torch.equal(runs[0][2], pool.arena), "attend_tc arena writes not deterministic"
    del arena0, runs[0]
    out, probs = runs[-1][0].cpu().numpy(), runs[-1][1].cpu().numpy()
    snap = dict(pages=v["pages"], table=v["table"], n_h=v["n_h"], n_l=v["n_l"], seq_len=v["seq_len"],
                win_k=v["win_k"], win_v=v["win_v"])
    eq1.check_units(snap, geom, L, W, d, LyH, q, out, probs, sample, where="fullsize tc")
    # the significance written back (Q33): (s * c + a) / (c + 1), c = N - 2 - pos, a = the float64 score
    N = T
    for u in sample:
        k_, v_, pos = eq1.unit_tokens64(v["pages"], v["table"][u].cpu().numpy(), int(v["n_h"][u]), int(v["n_l"][u]),
                                        N, v["win_k"][u].cpu().numpy(), v["win_v"][u].cpu().numpy(), geom, L, W, d)
        _, a = eq1.attend64(q[u], k_, v_)
        aft = _unit_scores(v, geom, L, u)
        for i, ps in enumerate(pos[:len(aft)]):
            s0, s1 = before[u][int(ps)], aft[int(ps)]
            cc = N - 2 - int(ps)
            want = (s0 * cc + float(a[i])) / (cc + 1) if cc >= 0 else s0
            assert abs(s1 - want) <= 1e-4 * max(abs(want), 1e-6), (u, ps, s1, want)


def _unit_scores(v, geom, L, u):
    """{position: significance} of unit u's stored tokens, read from the pool's pages"""
    out = {}
    table = v["table"][u].cpu().numpy()
    for cls, n in ((1, int(v["n_h"][u])), (2, int(v["n_l"][u]))):
        g = geom[cls]
        C = g["C"]
        npg = -(-n // C)
        cols = np.arange(npg) if cls == 1 else L - 1 - np.arange(npg)
        pids = torch.from_numpy(table[cols].astype(np.int64)).to(v["pages"].device)
        pg = v["pages"][pids].cpu().numpy()
        sc = np.ascontiguousarray(pg[:, g["off_score"]:g["off_score"] + 4 * C]).view(np.float32).reshape(-1)[:n]
        ps = np.ascontiguousarray(pg[:, g["off_pos"]:g["off_pos"] + 4 * C]).view(np.int32).reshape(-1)[:n]
        out.update({int(p): float(s) for p, s in zip(ps, sc)})
    return out
