"""Seeded synthetic inputs shaped like the paper's workloads (DESIGN.md §5 "input recipe").

This module holds NONE of the method's arithmetic: it only draws inputs (significance values, K/V
vectors, per-unit class mixes, significance drift standing in for attention updates) and is shared by the
oracle side and the CUDA side of every test and of bench.py.  Everything is counter-based (splitmix64
over (seed, stream, global unit, position, element)) and built from integer ops plus single IEEE fp32
operations, so a CPU tensor and a CUDA tensor drawn for the same counters are bit-identical and a
sample of units can be regenerated on the host one by one.

Global unit index: ug = (r * Ly + l) * H_total + h with h the GLOBAL KV head, so the data a unit sees is
the same at any GPU count (PIN-13).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


_C1 = _s64(0x9E3779B97F4A7C15)
_C2 = _s64(0xBF58476D1CE4E5B9)
_C3 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, s: int) -> torch.Tensor:
    return (x >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors with wrapping arithmetic (two's complement)."""
    z = x + _C1
    z = (z ^ _lsr(z, 30)) * _C2
    z = (z ^ _lsr(z, 27)) * _C3
    return z ^ _lsr(z, 31)


def splitmix64_int(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    return _s64(splitmix64_int((seed << 8) ^ stream ^ 0x5DEECE66D))


S_KEY, S_VAL, S_SIG_PREFILL, S_SIG_DECODE, S_NEW_K, S_NEW_V, S_DRIFT, S_MIX = range(8)


def hash_ctr(seed: int, stream: int, ctr: torch.Tensor) -> torch.Tensor:
    return splitmix64(ctr ^ stream_key(seed, stream))


def _bits(h: torch.Tensor, lo: int, n: int) -> torch.Tensor:
    return (h >> lo) & ((1 << n) - 1)


# ------------------------------------------------------------------------------------------- geometry
@dataclass(frozen=True)
class Shape:
    """Unit shape of a pool shard: R requests x Ly layers x heads [h0, h0 + H) of H_total."""
    R: int
    Ly: int
    H: int
    H_total: int | None = None
    h0: int = 0
    req_ids: tuple | None = None      # global request id of each local request slot (default: identity)

    @property
    def Ht(self) -> int:
        return self.H if self.H_total is None else self.H_total

    @property
    def U(self) -> int:
        return self.R * self.Ly * self.H

    def global_units(self, reqs, device="cpu") -> torch.Tensor:
        """[len(reqs), Ly*H] int64 global unit ids for local request ids `reqs`, local (l, h) order."""
        rr = np.asarray(reqs, dtype=np.int64)
        if self.req_ids is not None:
            rr = np.asarray(self.req_ids, dtype=np.int64)[rr]
        r = torch.as_tensor(rr, device=device).view(-1, 1, 1)
        l = torch.arange(self.Ly, device=device, dtype=torch.int64).view(1, -1, 1)
        h = torch.arange(self.H, device=device, dtype=torch.int64).view(1, 1, -1) + self.h0
        return ((r * self.Ly + l) * self.Ht + h).reshape(len(reqs), self.Ly * self.H)


# ------------------------------------------------------------------------------------------- K / V
def kv_values(seed: int, stream: int, ug: torch.Tensor, t0: int, T: int, d: int) -> torch.Tensor:
    """fp16 [*ug.shape, T, d]: triangular(-4, 4) values — the sum of two 16-bit uniforms, exact in fp32,
    scaled by 2^-14 and converted round-to-nearest-even."""
    dev = ug.device
    t = torch.arange(t0, t0 + T, device=dev, dtype=torch.int64)
    e = torch.arange(d, device=dev, dtype=torch.int64)
    ctr = ((ug.unsqueeze(-1).unsqueeze(-1) << 21) + t.view(-1, 1)) * d + e      # [..., T, d]
    h = hash_ctr(seed, stream, ctr >> 1)
    half = torch.where((ctr & 1) == 1, _bits(h, 32, 32), _bits(h, 0, 32))
    x = (_bits(half, 0, 16) + _bits(half, 16, 16) - 65535).to(torch.float32) * (2.0 ** -14)
    return x.to(torch.float16)


# ------------------------------------------------------------------------------------------- class mix
def unit_mix(seed: int, ug: torch.Tensor, mix=(0.35, 0.45, 0.20), Ly: int = 1, Ht: int = 1):
    """Per-unit target class mix as integer thresholds over 2^24 (High: x < th_h; Low: th_h <= x < th_l).

    Per-head and per-request dynamic sparsity: base mix, a per-layer shift, and a per-unit
    jitter of +-0.15, drawn from integer hashes and renormalised in float64 (host-side, tiny)."""
    ugn = ug.detach().cpu().numpy().astype(np.int64).ravel()
    out_h = np.empty(ugn.shape, np.int64)
    out_l = np.empty(ugn.shape, np.int64)
    key = stream_key(seed, S_MIX)
    for i, g in enumerate(ugn):
        hv = splitmix64_int((int(g) ^ key) & _M64)
        layer = (int(g) // Ht) % Ly
        lv = splitmix64_int((layer ^ key ^ 0xABCDEF) & _M64)
        w = []
        for k, base in enumerate(mix):
            jit = ((hv >> (16 * k)) & 0xFFFF) / 65535.0 - 0.5
            lsh = ((lv >> (16 * k)) & 0xFFFF) / 65535.0 - 0.5
            w.append(max(0.0, base * (1.0 + 0.6 * jit + 0.3 * lsh)) if base > 0 else 0.0)
        s = sum(w) or 1.0
        ph, pl = w[0] / s, w[1] / s
        out_h[i] = int(ph * (1 << 24))
        out_l[i] = int((ph + pl) * (1 << 24))
    sh = tuple(ug.shape)
    return (torch.from_numpy(out_h.reshape(sh)).to(ug.device), torch.from_numpy(out_l.reshape(sh)).to(ug.device))


def _sig_from_hash(h: torch.Tensor, th: torch.Tensor, tl: torch.Tensor, mix_h, mix_l) -> torch.Tensor:
    """Significance of a token whose target class is drawn against the unit mix:
    High: th*(1+2u); Low: tl + (th-tl)*u (kept < th); Pruned: tl*u; plus exact-threshold snaps (pin Q2),
    a small lattice of exact powers of two shared by many tokens (ties, pin Q6) and signed zeros."""
    x = _bits(h, 0, 24)
    u = _bits(h, 24, 23).to(torch.float32) * (2.0 ** -23)                       # exact, [0, 1)
    sp = _bits(h, 47, 8)                                                         # special draw
    one = torch.ones_like(u)
    hi = th * (one + u * 2.0)
    lo = tl + (th - tl) * u
    lo = torch.where(lo >= th, tl, lo)
    pr = tl * u
    s = torch.where(x < mix_h, hi, torch.where(x < mix_l, lo, pr))
    lat_tab = torch.tensor([2.0 ** -k for k in range(6, 14)], dtype=torch.float32, device=h.device)
    lattice = lat_tab[_bits(h, 55, 3)]                                           # 2^-6 .. 2^-13, exact
    s = torch.where(sp < 3, th, s)                  # ~1.2% snapped onto theta_h
    s = torch.where((sp >= 3) & (sp < 6), tl, s)    # ~1.2% snapped onto theta_l
    s = torch.where((sp >= 6) & (sp < 10), lattice, s)
    s = torch.where(sp == 10, torch.zeros_like(s), s)
    s = torch.where(sp == 11, torch.full_like(s, -0.0), s)
    return s


def prefill_sig(seed: int, ug: torch.Tensor, T: int, alpha_h: float, alpha_l: float, mix_h, mix_l,
                lens=None, denominator: int = 0) -> torch.Tensor:
    """fp32 [*ug.shape, T] prompt significance drawn relative to the §4 thresholds alpha/i (or alpha/n)."""
    dev = ug.device
    t = torch.arange(T, device=dev, dtype=torch.int64)
    ctr = (ug.unsqueeze(-1) << 24) + t
    h = hash_ctr(seed, S_SIG_PREFILL, ctr)
    if denominator == 0:
        den = (t + 1).to(torch.float32).expand(h.shape)
    else:
        den = torch.as_tensor(lens, device=dev).to(torch.float32).view(-1, *([1] * (ug.dim()))).expand(h.shape)
    ah = torch.tensor(alpha_h, dtype=torch.float32, device=dev)
    al = torch.tensor(alpha_l, dtype=torch.float32, device=dev)
    th, tl = ah / den, al / den
    return _sig_from_hash(h, th, tl, mix_h.unsqueeze(-1), mix_l.unsqueeze(-1))


def decode_sig(seed: int, ug: torch.Tensor, N: torch.Tensor, W: int, alpha_h: float, alpha_l: float,
               mix_h, mix_l) -> torch.Tensor:
    """fp32 cand_sig for each unit's t_c (position N-1-W) relative to alpha/N (Algorithm 1)."""
    dev = ug.device
    pc = (N - 1 - W).clamp(min=0).to(torch.int64)
    h = hash_ctr(seed, S_SIG_DECODE, (ug << 24) + pc)
    den = N.to(torch.float32).clamp(min=1.0)
    ah = torch.tensor(alpha_h, dtype=torch.float32, device=dev)
    al = torch.tensor(alpha_l, dtype=torch.float32, device=dev)
    return _sig_from_hash(h, ah / den, al / den, mix_h, mix_l)


def new_token_kv(seed: int, ug: torch.Tensor, pos: torch.Tensor, d: int):
    """fp16 [U, d] K and V of the token appended at position `pos` (per unit)."""
    dev = ug.device
    e = torch.arange(d, device=dev, dtype=torch.int64)
    out = []
    for stream in (S_NEW_K, S_NEW_V):
        ctr = (((ug << 21) + pos.to(torch.int64)).unsqueeze(-1)) * d + e
        h = hash_ctr(seed, stream, ctr >> 1)
        half = torch.where((ctr & 1) == 1, _bits(h, 32, 32), _bits(h, 0, 32))
        x = (_bits(half, 0, 16) + _bits(half, 16, 16) - 65535).to(torch.float32) * (2.0 ** -14)
        out.append(x.to(torch.float16))
    return out[0], out[1]


# ------------------------------------------------------------------------------------------- drift
_DRIFT = (0.5, 0.75, 1.0, 1.0, 1.0, 1.0, 1.25, 2.0)


def drift_factor(seed: int, step: int, ug: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
    """Multiplier in {0.5, 0.75, 1, 1.25, 2} keyed by (unit, position, step): stands in for the attention
    epilogue's significance update between decode steps (Q5; out of scope, NEXT-2)."""
    h = hash_ctr(seed ^ (step << 20), S_DRIFT, (ug.to(torch.int64) << 24) + pos.to(torch.int64))
    tab = torch.tensor(_DRIFT, dtype=torch.float32, device=ug.device)
    return tab[_bits(h, 0, 3)]


def apply_drift(seed: int, step: int, shape: Shape, pages_u8: torch.Tensor, table: torch.Tensor,
                n_h: torch.Tensor, n_l: torch.Tensor, geom: dict, L: int, active_units=None, chunk: int = 1 << 22,
                ttable=None, n_t=None):
    """sig <- sig * m (one fp32 multiply) for every stored token of every unit, in place on page bytes.

    `pages_u8` is a contiguous uint8 [P, page_bytes] tensor (oracle numpy view via torch.from_numpy, or
    the CUDA arena); `geom` = {cls: (C, off_score, off_pos)} for cls 1 (high) and 2 (low), and 4 (the NEXT-4
    FP16 tier, pages in `ttable` with `n_t` tokens) when given.  Pure harness: stands in for the attention
    epilogue."""
    dev = pages_u8.device
    U = table.shape[0]
    pb = pages_u8.shape[1]
    words_f = pages_u8.view(-1).view(torch.float32)
    words_i = pages_u8.view(-1).view(torch.int32)
    ug_all = shape.global_units(list(range(shape.R)), device=dev).reshape(-1)
    table = table.to(dev)
    secs = ((1, n_h), (2, n_l)) + (((4, n_t),) if ttable is not None else ())
    for cls, n in secs:
        C, off_s, off_p = geom[cls]
        n64 = n.to(dev).to(torch.int64)
        if active_units is not None:
            n64 = torch.where(active_units.to(dev), n64, torch.zeros_like(n64))
        npg = (n64 + C - 1) // C
        maxp = int(npg.max().item()) if U else 0
        if maxp == 0:
            continue
        # one row per (unit, page) — then C slots per page
        kk = torch.arange(maxp, device=dev, dtype=torch.int64)
        vp = kk.view(1, -1) < npg.view(-1, 1)
        uu, pk = vp.nonzero(as_tuple=True)
        for a in range(0, uu.numel(), chunk):
            u1, p1 = uu[a:a + chunk], pk[a:a + chunk]
            col = p1 if cls != 2 else (L - 1 - p1)
            pid = (ttable.to(dev) if cls == 4 else table)[u1, col].to(torch.int64)
            idx = torch.arange(C, device=dev, dtype=torch.int64).view(1, -1)
            slot = p1.view(-1, 1) * C + idx
            ok = slot < n64[u1].view(-1, 1)
            wbase = (pid * pb).view(-1, 1) // 4
            ws = (wbase + off_s // 4 + idx)[ok]
            wp = (wbase + off_p // 4 + idx)[ok]
            uv = u1.view(-1, 1).expand(-1, C)[ok]
            f = drift_factor(seed, step, ug_all[uv], words_i[wp])
            words_f[ws] = words_f[ws] * f
