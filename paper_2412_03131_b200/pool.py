"""Pool: a torch-owned arena plus the C-ABI handle (plumbing only — every step runs in libdkv.so).

torch supplies the device memory (one uint8 CUDA tensor, the arena) and the stream; the methods call
the C ABI by name.  ``views()`` exposes the arena's buffers as torch views at the offsets the library
reports (dkv_pool_layout) for inspection by tests and the admission logic.
"""
from __future__ import annotations

import numpy as np
import torch

from . import dkv as _d


class Pool:
    def __init__(self, cfg: _d.dkv_config_t, device=None, stream=None):
        self.cfg = cfg
        self.layout = _d.dkv_pool_layout(cfg)
        self.device = torch.device(device if device is not None else "cuda")
        nbytes = int(self.layout.arena_bytes)
        self.arena = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.stream = stream
        self.handle = _d.dkv_pool_init(cfg, self.arena, nbytes, stream)
        L = self.layout
        self.U, self.L, self.page_bytes = L.units, L.table_len, L.page_bytes
        self.LyH = cfg.num_layers * cfg.num_kv_heads

    def close(self):
        if getattr(self, "handle", None):
            _d.dkv_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the ABI, by name
    def classify_decode(self, sig, dec, stream=None):
        return _d.dkv_classify(self.handle, _d.DKV_PHASE_DECODE, None, None, 0, sig, 0, dec, None,
                               stream or self.stream)

    def classify_prefill(self, reqs, lens, sig, token_class=None, stream=None):
        return _d.dkv_classify(self.handle, _d.DKV_PHASE_PREFILL, reqs, lens, len(reqs), sig, sig.shape[-1], None,
                               token_class, stream or self.stream)

    def compact_alloc(self, dec=None, stream=None):
        return _d.dkv_compact_alloc(self.handle, dec, stream or self.stream)

    def quant_write_decode(self, dec, k, v, sig, stream=None):
        return _d.dkv_quant_write(self.handle, _d.DKV_PHASE_DECODE, dec, k, v, 0, sig, 0, stream or self.stream)

    def decode_step_host(self, h_sig, h_kv, h_dec=None, stream=None):
        """The whole decode step from host buffers (dkv_decode_step_host): h_sig fp32 [U] or None, h_kv int16
        [2][U][d] (keys then values), h_dec int32 [U][4] or None — CPU tensors, pinned for async copies."""
        if getattr(self, "_stage", None) is None:
            self._stage_bytes = _d.dkv_decode_stage_bytes(self.handle)
            self._stage = torch.empty(self._stage_bytes, dtype=torch.uint8, device=self.device)
        return _d.dkv_decode_step_host(self.handle, h_sig, h_kv, h_dec, self._stage, self._stage_bytes,
                                       stream or self.stream)

    def decode_graph(self, steps, sig, k, v, dec, flags=_d.DKV_GRAPH_PDL):
        """dkv_decode_graph_create: `steps` decode steps captured as one CUDA graph.  sig fp32 [steps][U] (or
        [U] reused, or None: window significance), k / v int16 [steps][U][d] (or [U][d] reused), dec int32
        [U][4]: CUDA tensors that must outlive the graph.  Returns a DecodeGraph."""
        U, d = self.U, self.cfg.head_dim
        sig_step = U if (sig is not None and sig.dim() == 2) else 0
        kv_step = U * d if k.dim() == 3 else 0
        h = _d.dkv_decode_graph_create(self.handle, steps, sig, sig_step, k, v, kv_step, dec, flags)
        return DecodeGraph(h, steps, (sig, k, v, dec))

    def quant_write_prefill(self, k, v, sig, stream=None):
        return _d.dkv_quant_write(self.handle, _d.DKV_PHASE_PREFILL, None, k, v, k.shape[-2], sig, sig.shape[-1],
                                  stream or self.stream)

    def attend(self, q, out=None, probs=None, stream=None):
        """NEXT-2: q = fp16 (as int16) [U][q_per_kv][d] CUDA tensor; out fp32 [U][G][d] / probs fp32 [U][M] or None"""
        return _d.dkv_attend(self.handle, q, out, probs, stream or self.stream)

    def attend_tc(self, q, out=None, probs=None, stream=None):
        """NEXT-2 on tensor cores (dkv_attend_tc): same buffers as attend()"""
        return _d.dkv_attend_tc(self.handle, q, out, probs, stream or self.stream)

    AUDIT_KEYS = ("owned_twice", "unowned", "bad_slots", "used_pages", "free_pages", "dup_positions",
                  "positions_out_of_range", "over_capacity")

    def audit(self, stream=None):
        """dkv_audit: the pool's invariants checked on the device; returns a dict of AUDIT_KEYS (sound: all zero
        except used_pages + free_pages == num_pages).  Synchronises the stream."""
        s = stream or self.stream
        if getattr(self, "_audit_buf", None) is None:
            self._audit_buf = (torch.empty(int(self.cfg.num_pages), dtype=torch.int32, device=self.device),
                               torch.empty(8, dtype=torch.int64, device=self.device))
        hist, res = self._audit_buf
        _d.dkv_audit(self.handle, hist, res, s)
        torch.cuda.synchronize(self.device)
        vals = res.cpu().tolist()
        return dict(zip(self.AUDIT_KEYS, vals))

    def set_head_thresholds(self, alpha_h, alpha_l, stream=None):
        """NEXT-4: per-(layer, head) thresholds (host sequences of Ly*H floats), or None for the pool-wide pair"""
        return _d.dkv_set_head_thresholds(self.handle, alpha_h, alpha_l, stream or self.stream)

    def free(self, reqs, stream=None):
        return _d.dkv_free(self.handle, reqs, len(reqs), stream or self.stream)

    def query(self, stream=None):
        return _d.dkv_pool_query(self.handle, stream or self.stream)

    def new_decisions(self):
        return torch.empty((self.U, 4), dtype=torch.int32, device=self.device)

    # ---- views (plumbing for tests / admission)
    def _view(self, off, nbytes, dtype, shape):
        t = self.arena[int(off): int(off) + int(nbytes)]
        return t.view(dtype).view(shape)

    def views(self):
        L, c = self.layout, self.cfg
        U, R, P = self.U, c.max_requests, c.num_pages
        W, d = c.window, c.head_dim
        return dict(
            ctrl=self._view(L.off_ctrl, 32, torch.int64, (4,)),           # start, free, {status, oom}
            ring=self._view(L.off_ring, 4 * P, torch.int32, (P,)),
            table=self._view(L.off_table, 4 * U * self.L, torch.int32, (U, self.L)),
            n_h=self._view(L.off_n_h, 4 * U, torch.int32, (U,)),
            n_l=self._view(L.off_n_l, 4 * U, torch.int32, (U,)),
            req_state=self._view(L.off_req_state, R, torch.int8, (R,)),
            seq_len=self._view(L.off_seq_len, 4 * R, torch.int32, (R,)),
            win_k=self._view(L.off_win_k, 2 * U * W * d, torch.int16, (U, W, d)),
            win_v=self._view(L.off_win_v, 2 * U * W * d, torch.int16, (U, W, d)),
            pages=self._view(L.off_pages, P * self.page_bytes, torch.uint8, (P, self.page_bytes)),
            stats=self._view(L.off_stats, 32, torch.int64, (4,)),
            win_sig=self._view(L.off_win_sig, 4 * U * W, torch.float32, (U, W)),
            secmin=self._view(L.off_secmin, 32 * U, torch.int32, (U, 8)),
            ttable=self._view(L.off_ttable, 4 * U * L.table_len_top, torch.int32, (U, L.table_len_top)),   # NEXT-4
            n_t=self._view(L.off_n_t, 4 * U, torch.int32, (U,)),
        )

    def geom(self):
        L, cf = self.layout, self.cfg
        bits = {1: (cf.kbits_high, cf.vbits_high), 2: (cf.kbits_low, cf.vbits_low)}
        g = {c: dict(C=L.C[c], kbits=bits[c][0], vbits=bits[c][1], k_row=L.k_row[c], v_row=L.v_row[c], off_k=L.off_k[c], off_kmeta=L.off_kmeta[c],
                     off_v=L.off_v[c], off_vmeta=L.off_vmeta[c], off_score=L.off_score[c], off_pos=L.off_pos[c])
             for c in (1, 2)}
        if cf.top_tier:                                  # NEXT-4 TOP pages: fp16 rows, no metadata
            g[4] = dict(C=L.C_top, kbits=16, vbits=16, k_row=L.row_top, v_row=L.row_top, off_k=L.off_k_top,
                        off_kmeta=L.off_k_top + L.C_top * L.row_top, off_v=L.off_v_top,
                        off_vmeta=L.off_v_top + L.C_top * L.row_top, off_score=L.off_score_top, off_pos=L.off_pos_top)
        return g


class DecodeGraph:
    """A captured decode-step graph (keeps its buffers alive); launch() replays it on the current stream."""

    def __init__(self, handle, steps, buffers):
        self.handle, self.steps, self._buffers = handle, steps, buffers

    def launch(self, stream=None):
        return _d.dkv_decode_graph_launch(self.handle, stream)

    def kernel_ms(self):
        """[steps][3] classify / compact_alloc / quant_write ms of the last replay (DKV_GRAPH_EVENTS graphs)"""
        return _d.dkv_decode_graph_kernel_ms(self.handle, self.steps)

    def close(self):
        if getattr(self, "handle", None):
            _d.dkv_decode_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decisions_to_numpy(dec: torch.Tensor) -> np.ndarray:
    return dec.detach().cpu().contiguous().numpy().view(_d.DECISION_DTYPE).reshape(-1)
