"""Harness backend driving the CUDA C-ABI (paper_2412_03131_b200) with the same calls as OracleBackend."""
from __future__ import annotations

import numpy as np
import torch

import synth
from paper_2412_03131_b200 import Pool, decisions_to_numpy
from paper_2412_03131_b200 import dkv as D


class GpuBackend:
    name = "gpu"

    def __init__(self, scn, device="cuda"):
        self.scn = scn
        cfg = D.make_config(scn.R, scn.Ly, scn.H, scn.d, scn.M, scn.W, scn.Ch, scn.Cl, scn.kbh, scn.vbh, scn.kbl,
                            scn.vbl, scn.P, scn.alpha_h, scn.alpha_l, scn.prompt_denominator, scn.tile_units,
                            scn.prefill_workflow, scn.q_per_kv, scn.top_tier, scn.alpha_t, scn.Ct)
        self.pool = Pool(cfg, device=device)
        self.U, self.L, self.page_bytes = self.pool.U, self.pool.L, self.pool.page_bytes
        self.v = self.pool.views()
        self.geom = self.pool.geom()
        self.dec = self.pool.new_decisions()
        self.device = device

    def _cuda(self, x):
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(x)
        return x.to(self.device).contiguous()

    def classify_decode(self, cand):
        self._cand = None if cand is None else self._cuda(cand.float() if isinstance(cand, torch.Tensor) else cand)
        self.pool.classify_decode(self._cand, self.dec)
        return 0, self.dec

    def classify_prefill(self, reqs, lens, sig):
        self._sig = self._cuda(sig)
        self.pool.classify_prefill(list(reqs), list(lens), self._sig)
        return 0

    def compact_alloc(self, dec):
        self.pool.compact_alloc(dec if isinstance(dec, torch.Tensor) else None)
        return 0

    def quant_write_decode(self, dec, k, v, cand):
        k, v = self._cuda(k).view(torch.int16), self._cuda(v).view(torch.int16)
        self.pool.quant_write_decode(dec, k, v, None if cand is None else self._cuda(cand))
        return 0

    def set_head_thresholds(self, ah, al):
        self.pool.set_head_thresholds(ah, al)
        return 0

    def attend(self, q, want_out=True, want_probs=False):
        G, d, M = self.scn.q_per_kv, self.scn.d, self.scn.M
        qd = self._cuda(np.ascontiguousarray(q).view(np.int16))
        out = torch.zeros((self.U, G, d), dtype=torch.float32, device=self.device) if want_out else None
        probs = torch.zeros((self.U, M), dtype=torch.float32, device=self.device) if want_probs else None
        self.pool.attend(qd, out, probs)
        torch.cuda.synchronize()
        return 0, (out.cpu().numpy() if want_out else None), (probs.cpu().numpy() if want_probs else None)

    def attend_tc(self, q, want_out=True, want_probs=False):
        """NEXT-2 on tensor cores (dkv_attend_tc); same buffers as attend()"""
        G, d, M = self.scn.q_per_kv, self.scn.d, self.scn.M
        qd = self._cuda(np.ascontiguousarray(q).view(np.int16))
        out = torch.zeros((self.U, G, d), dtype=torch.float32, device=self.device) if want_out else None
        probs = torch.zeros((self.U, M), dtype=torch.float32, device=self.device) if want_probs else None
        self.pool.attend_tc(qd, out, probs)
        torch.cuda.synchronize()
        return 0, (out.cpu().numpy() if want_out else None), (probs.cpu().numpy() if want_probs else None)

    def quant_write_prefill(self, k, v, sig):
        k, v = self._cuda(k).view(torch.int16), self._cuda(v).view(torch.int16)
        self.pool.quant_write_prefill(k, v, self._cuda(sig))
        return 0

    def free(self, reqs):
        self.pool.free(list(reqs))
        return 0

    def take_status(self):
        st, _ = self.pool.query()
        return st

    def drift(self, step):
        v = self.v
        top = self.scn.top_tier
        synth.apply_drift(self.scn.seed, step, self.scn.shape, v["pages"], v["table"], v["n_h"], v["n_l"],
                          {c: (self.geom[c]["C"], self.geom[c]["off_score"], self.geom[c]["off_pos"]) for c in self.geom},
                          self.L, ttable=v["ttable"] if top else None, n_t=v["n_t"] if top else None)

    def snapshot(self, pages=True):
        torch.cuda.synchronize()
        v = self.v
        ctrl = v["ctrl"].cpu().numpy()
        s = dict(ring=v["ring"].cpu().numpy(), start=int(ctrl[0]), free=int(ctrl[1]),
                 status=int(ctrl[2] & 0xFFFFFFFF), table=v["table"].cpu().numpy(), n_h=v["n_h"].cpu().numpy(),
                 n_l=v["n_l"].cpu().numpy(), req_state=v["req_state"].cpu().numpy(),
                 seq_len=v["seq_len"].cpu().numpy(), win_k=v["win_k"].cpu().numpy().view(np.uint16),
                 win_v=v["win_v"].cpu().numpy().view(np.uint16), win_sig=v["win_sig"].cpu().numpy())
        if self.scn.top_tier:
            s.update(ttable=v["ttable"].cpu().numpy(), n_t=v["n_t"].cpu().numpy())
        if pages:
            s["pages"] = v["pages"].cpu().numpy()
        return s


def dec_np(dec):
    if isinstance(dec, torch.Tensor):
        return decisions_to_numpy(dec)
    return dec


def compare_state(a, b, keys=("ring", "start", "free", "table", "n_h", "n_l", "req_state", "seq_len", "win_k", "win_v",
                              "win_sig", "ttable", "n_t",
                              "pages"), where=""):
    for k in keys:
        if k not in a or k not in b:
            continue
        x, y = a[k], b[k]
        if isinstance(x, np.ndarray):
            if not np.array_equal(x, y):
                bad = np.argwhere(x != y)
                raise AssertionError(f"[{where}] {k} differs at {len(bad)} positions, first {bad[:5].tolist()}: "
                                     f"oracle {x[tuple(bad[0])]} vs gpu {y[tuple(bad[0])]}")
        elif x != y:
            raise AssertionError(f"[{where}] {k}: oracle {x} vs gpu {y}")
