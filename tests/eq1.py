"""Independent float64 evaluation of the paper's attention (Eq. 1) over a pool's compressed cache,
with the GQA score = max over the query heads of a group.  Test infrastructure: it reads the page
bytes itself (codes LSB-first, Q17; fp16 {s, z} metadata; X^ = s*Q + z) and shares nothing with the
oracle's or the kernels' arithmetic, so a GPU attention result can be pinned to the paper's formula directly
instead of to another implementation.

Token order (reading Q31): high slots, low slots, then the FP16 window oldest first."""
from __future__ import annotations

import math

import numpy as np


def _unpack_rows(codes: np.ndarray, bits: int, d: int) -> np.ndarray:
    """codes u8 [n, d*bits/8] -> float64 [n, d] code values (element e in bits [e*bits, (e+1)*bits))"""
    b = np.unpackbits(codes.astype(np.uint8), axis=1, bitorder="little")          # [n, d*bits]
    vals = b.reshape(codes.shape[0], d, bits) @ (1 << np.arange(bits))
    return vals.astype(np.float64)


def unit_tokens64(pages, table_row, n_h, n_l, seq_len, win_k_u, win_v_u, geom, L, W, d):
    """(keys, values, positions) of one unit in Q31 order, float64.  `pages` is a host array [P, page_bytes]
    or a torch tensor (only the unit's pages are fetched); `geom` maps class 1/2 to a dict with C, kbits,
    vbits, k_row, v_row and the segment offsets; win_k_u / win_v_u are the unit's [W, d] window rows as
    uint16 (fp16 bits)."""
    ks, vs, ps = [], [], []
    for cls, n in ((1, int(n_h)), (2, int(n_l))):
        if n == 0:
            continue
        g = geom[cls]
        C = g["C"]
        npg = -(-n // C)
        cols = np.arange(npg) if cls == 1 else L - 1 - np.arange(npg)
        pids = np.asarray(table_row)[cols].astype(np.int64)
        if type(pages).__module__.startswith("torch"):
            import torch
            pg = pages[torch.from_numpy(pids).to(pages.device)].cpu().numpy()
        else:
            pg = np.asarray(pages)[pids]
        for off, row, meta, bits, acc in ((g["off_k"], g["k_row"], g["off_kmeta"], g["kbits"], ks),
                                          (g["off_v"], g["v_row"], g["off_vmeta"], g["vbits"], vs)):
            codes = pg[:, off:off + C * row].reshape(npg * C, row)[:n]
            m = np.ascontiguousarray(pg[:, meta:meta + 4 * C]).view(np.float16).reshape(npg * C, 2)[:n]
            acc.append(m[:, :1].astype(np.float64) * _unpack_rows(codes, bits, d) + m[:, 1:].astype(np.float64))
        ps.append(np.ascontiguousarray(pg[:, g["off_pos"]:g["off_pos"] + 4 * C]).view(np.int32).reshape(-1)[:n])
    N = int(seq_len)
    wpos = np.arange(max(N - W, 0), N)
    if len(wpos):
        ks.append(np.asarray(win_k_u)[wpos % W].view(np.float16).astype(np.float64))
        vs.append(np.asarray(win_v_u)[wpos % W].view(np.float16).astype(np.float64))
        ps.append(wpos.astype(np.int32))
    if not ks:
        return np.zeros((0, d)), np.zeros((0, d)), np.zeros(0, np.int32)
    return np.concatenate(ks), np.concatenate(vs), np.concatenate(ps)


def attend64(q_u: np.ndarray, keys: np.ndarray, values: np.ndarray):
    """Eq. 1 for the G query heads of one unit: out [G, d] = softmax(q k^T / sqrt(d)) v; scores [n] = max over
    the G heads of the attention weights."""
    d = q_u.shape[-1]
    if keys.shape[0] == 0:
        return np.zeros((q_u.shape[0], d)), np.zeros(0)
    logits = (q_u.astype(np.float64) @ keys.T) / math.sqrt(d)
    a = np.exp(logits - logits.max(axis=1, keepdims=True))
    a /= a.sum(axis=1, keepdims=True)
    return a @ values, a.max(axis=0)


def check_units(snap, geom, L, W, d, LyH, q, out, probs, units, rtol=2e-4, atol=2e-5, prtol=2e-5, patol=1e-7,
                where=""):
    """Compare a GPU attention result (out [U, G, d], probs [U, M] or None) for `units` against Eq. 1 evaluated
    in float64 from the snapshot `snap` (pages, table, n_h, n_l, seq_len, win_k, win_v as host arrays or device
    tensors).  Returns the largest relative output error seen."""
    worst = 0.0
    for u in units:
        r = u // LyH
        k, v, pos = unit_tokens64(snap["pages"], _row(snap["table"], u), _at(snap["n_h"], u), _at(snap["n_l"], u),
                                  _at(snap["seq_len"], r), _row(snap["win_k"], u), _row(snap["win_v"], u),
                                  geom, L, W, d)
        if len(pos) == 0:
            continue
        ref_out, ref_p = attend64(q[u], k, v)
        got = np.asarray(out[u], np.float64)
        err = np.abs(got - ref_out)
        assert (err <= atol + rtol * np.abs(ref_out)).all(), \
            f"[{where}] unit {u}: attention output off Eq. 1 by {float(err.max())}"
        worst = max(worst, float((err / (np.abs(ref_out) + atol / rtol)).max()))
        if probs is not None:
            gp = np.asarray(probs[u][:len(pos)], np.float64)
            assert np.allclose(gp, ref_p, rtol=prtol, atol=patol), f"[{where}] unit {u}: scores off Eq. 1"
    return worst


def _row(x, u):
    r = x[u]
    return r.cpu().numpy() if type(r).__module__.startswith("torch") else np.asarray(r)


def _at(x, i):
    r = x[i]
    return int(r.item() if hasattr(r, "item") else r)
