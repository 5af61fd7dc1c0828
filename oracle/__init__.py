"""Serial CPU oracle for DiffKV's KV memory manager (arXiv 2412.03131) — ctypes wrapper.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
(``paper_2412_03131_b200``) never imports it, and this package imports nothing from the product.

The arithmetic lives in ``dkv_oracle.c`` (plain serial C, ``-O2 -ffp-contract=off``); this module only
marshals numpy arrays and exposes the oracle's state as numpy views for comparison.

Parity status of each function:
  orc_f16_from_f32 / f32_from_f16   pinned: numpy.float16 over all binary16 values + random fp32 bits
  orc_quantize / dequantize         pinned: P:175-177 closed forms (grid, constant, error bound, range,
                                    monotone, 2^k invariance, idempotence)
  orc_geometry / table_bytes        pinned: P:500 32 MiB, Fig. 1 payload accounting
  orc_classify_decode               pinned: literal set-based Algorithm 1 in tests, PIN-5/6/7
  orc_classify_prefill              pinned: §4 thresholds brute force, PIN-6/7
  orc_compact_alloc                 pinned: Fig. 5 ring/table replay, invariants I1-I5,
                                    itertools.accumulate scan, PagedAttention reduction (PIN-6)
  orc_quant_write_*                 pinned: decoded codes vs orc_quantize of the generator's inputs
  orc_prefill_conservative          pinned: Fig. 5
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "dkv_oracle.c")
_HDR = os.path.join(_HERE, "dkv_oracle.h")
_lock = threading.Lock()

OK, ERR_INVALID, ERR_STATE, ERR_OOM, ERR_NONFINITE, ERR_OVERFLOW = 0, -1, -2, -3, -4, -5
DECODE, PREFILL = 0, 1
CLS_NONE, CLS_HIGH, CLS_LOW, CLS_PRUNED, CLS_TOP = 0, 1, 2, 3, 4
V_NONE, V_KEEP, V_DOWN, V_PRUNE = 0, 1, 2, 3
GROW_NONE, GROW_HIGH, GROW_LOW, GROW_TOP = 0, 1, 2, 3
REQ_IDLE, REQ_ADMITTING, REQ_ACTIVE, REQ_PENDING_FREE = 0, 1, 2, 3

DECISION_DTYPE = np.dtype([("tc_class", "u1"), ("v_action", "u1"), ("grow", "u1"), ("demand", "u1"),
                           ("v_slot", "<i4"), ("tc_slot", "<i4"), ("v_dst_slot", "<i4")])
assert DECISION_DTYPE.itemsize == 16


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, -O2 -ffp-contract=off, no fast-math)."""
    with _lock:
        stale = (not os.path.exists(_SO) or
                 os.path.getmtime(_SO) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
        if force or stale:
            tmp = _SO + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                                   "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _SO)
    return _SO


class Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("R", "Ly", "H", "d", "M", "W", "Ch", "Cl", "kbh", "vbh", "kbl", "vbl", "P")] + \
               [("alpha_h", C.c_float), ("alpha_l", C.c_float), ("prompt_denominator", C.c_int32),
                ("prefill_workflow", C.c_int32), ("q_per_kv", C.c_int32),
                ("top_tier", C.c_int32), ("alpha_t", C.c_float), ("Ct", C.c_int32)]


class ClassGeom(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("C", "kbits", "vbits", "k_row", "v_row", "off_k", "off_kmeta", "off_v",
                                          "off_vmeta", "off_score", "off_pos", "end")]


class _Pool(C.Structure):
    _fields_ = [("c", Config), ("U", C.c_int32), ("L", C.c_int32), ("page_bytes", C.c_int32),
                ("g", ClassGeom * 5),
                ("ring", C.POINTER(C.c_int32)), ("start", C.c_int64), ("free", C.c_int64),
                ("table", C.POINTER(C.c_int32)), ("n_h", C.POINTER(C.c_int32)), ("n_l", C.POINTER(C.c_int32)),
                ("req_state", C.POINTER(C.c_int8)), ("seq_len", C.POINTER(C.c_int32)),
                ("prompt_len", C.POINTER(C.c_int32)), ("pages", C.POINTER(C.c_uint8)),
                ("win_k", C.POINTER(C.c_uint16)), ("win_v", C.POINTER(C.c_uint16)),
                ("pf_nh", C.POINTER(C.c_int32)), ("pf_nl", C.POINTER(C.c_int32)),
                ("admit_list", C.POINTER(C.c_int32)), ("n_admit", C.c_int32),
                ("status", C.c_int32), ("last_phase", C.c_int32),
                ("last_demand", C.c_int64), ("last_freed", C.c_int64), ("oom_count", C.c_int32),
                ("last_reclaimed", C.c_int64), ("win_sig", C.POINTER(C.c_float)),
                ("head_ah", C.POINTER(C.c_float)), ("head_al", C.POINTER(C.c_float)), ("use_head", C.c_int32),
                ("Lt", C.c_int32), ("ttable", C.POINTER(C.c_int32)), ("n_t", C.POINTER(C.c_int32)),
                ("pf_nt", C.POINTER(C.c_int32))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        L.orc_f16_from_f32.argtypes = [C.c_float]; L.orc_f16_from_f32.restype = C.c_uint16
        L.orc_f32_from_f16.argtypes = [C.c_uint16]; L.orc_f32_from_f16.restype = C.c_float
        L.orc_f16_from_f32_array.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_f16_from_f32_array.restype = None
        L.orc_quantize.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, P(C.c_uint16), P(C.c_uint16)]
        L.orc_quantize.restype = C.c_int32
        L.orc_dequantize.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_uint16, C.c_uint16, C.c_void_p]
        L.orc_dequantize.restype = None
        L.orc_geometry.argtypes = [P(Config), P(C.c_int32), P(C.c_int32), P(C.c_int32), P(ClassGeom), P(ClassGeom)]
        L.orc_geometry.restype = C.c_int32
        L.orc_table_bytes.argtypes = [C.c_int64] * 4; L.orc_table_bytes.restype = C.c_int64
        L.orc_pool_new.argtypes = [P(Config)]; L.orc_pool_new.restype = P(_Pool)
        L.orc_pool_delete.argtypes = [P(_Pool)]; L.orc_pool_delete.restype = None
        L.orc_classify_decode.argtypes = [P(_Pool), C.c_void_p, C.c_void_p]
        L.orc_classify_prefill.argtypes = [P(_Pool), C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_compact_alloc.argtypes = [P(_Pool), C.c_void_p]
        L.orc_quant_write_decode.argtypes = [P(_Pool), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_quant_write_prefill.argtypes = [P(_Pool), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64]
        L.orc_free.argtypes = [P(_Pool), C.c_void_p, C.c_int32]
        L.orc_take_status.argtypes = [P(_Pool)]
        L.orc_prefill_conservative.argtypes = [P(_Pool), C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64,
                                               C.c_void_p, P(C.c_int64)]
        L.orc_attend.argtypes = [P(_Pool), C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_exp.argtypes = [C.c_float]; L.orc_exp.restype = C.c_float
        L.orc_set_head_thresholds.argtypes = [P(_Pool), C.c_void_p, C.c_void_p]
        L.orc_set_head_thresholds.restype = C.c_int32
        for f in ("orc_classify_decode", "orc_classify_prefill", "orc_compact_alloc", "orc_quant_write_decode",
                  "orc_quant_write_prefill", "orc_free", "orc_take_status", "orc_prefill_conservative", "orc_attend"):
            getattr(L, f).restype = C.c_int32
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------------------------- scalars
def f16_from_f32(x: float) -> int:
    return int(lib().orc_f16_from_f32(C.c_float(x)))


def f32_from_f16(h: int) -> float:
    return float(lib().orc_f32_from_f16(C.c_uint16(h)))


def f16_from_f32_array(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.zeros(x.shape, dtype=np.uint16)
    lib().orc_f16_from_f32_array(_ptr(x), _ptr(out), x.size)
    return out


def quantize(x, bits: int):
    """Quantize one vector.  Returns (status, packed codes uint8, s16 bits, z16 bits)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    d = x.shape[0]
    codes = np.zeros(max(1, d * bits // 8), dtype=np.uint8)
    s = C.c_uint16(0); z = C.c_uint16(0)
    st = lib().orc_quantize(_ptr(x), d, bits, _ptr(codes), C.byref(s), C.byref(z))
    return st, codes, s.value, z.value


def dequantize(codes, d: int, bits: int, s16: int, z16: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    out = np.zeros(d, dtype=np.float32)
    lib().orc_dequantize(_ptr(codes), d, bits, s16, z16, _ptr(out))
    return out


def unpack_codes(codes, d: int, bits: int) -> np.ndarray:
    """Unpack LSB-first packed codes (Q17) — plain bit arithmetic for tests."""
    codes = np.asarray(codes, dtype=np.uint8)
    idx = np.arange(d) * bits
    return ((codes[idx >> 3].astype(np.int32) >> (idx & 7)) & ((1 << bits) - 1)).astype(np.int32)


def make_config(**kw) -> Config:
    defaults = dict(R=4, Ly=2, H=4, d=64, M=128, W=16, Ch=16, Cl=32, kbh=8, vbh=4, kbl=4, vbl=2, P=1024,
                    alpha_h=1.0, alpha_l=0.02, prompt_denominator=0, prefill_workflow=0, q_per_kv=0,
                    top_tier=0, alpha_t=0.0, Ct=4)
    defaults.update(kw)
    return Config(**defaults)


def geometry(cfg: Config):
    U = C.c_int32(); L = C.c_int32(); pb = C.c_int32(); gh = ClassGeom(); gl = ClassGeom()
    st = lib().orc_geometry(C.byref(cfg), C.byref(U), C.byref(L), C.byref(pb), C.byref(gh), C.byref(gl))
    if st != OK:
        raise ValueError(f"invalid oracle config (status {st})")
    return dict(U=U.value, L=L.value, page_bytes=pb.value, high=gh, low=gl)


def table_bytes(batch, layers, kv_heads, L) -> int:
    return int(lib().orc_table_bytes(batch, layers, kv_heads, L))


# ---------------------------------------------------------------------------------------------- pool
class OraclePool:
    """Serial oracle pool.  State arrays are live numpy views of the C structure."""

    def __init__(self, cfg: Config | None = None, **kw):
        self.cfg = cfg if cfg is not None else make_config(**kw)
        self._p = lib().orc_pool_new(C.byref(self.cfg))
        if not self._p:
            raise ValueError("orc_pool_new failed (invalid config or out of host memory)")
        s = self._p.contents
        self.U, self.L, self.page_bytes = s.U, s.L, s.page_bytes
        self.geom = {CLS_HIGH: s.g[CLS_HIGH], CLS_LOW: s.g[CLS_LOW]}
        if self.cfg.top_tier:
            self.geom[CLS_TOP] = s.g[CLS_TOP]
        self.Lt = s.Lt
        c = self.cfg
        self.LyH = c.Ly * c.H

        def view(ptr, shape, dt):
            n = int(np.prod(shape))
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(dt)), shape=(max(n, 1),))[:n].reshape(shape)

        self.ring = view(s.ring, (c.P,), C.c_int32)
        self.table = view(s.table, (self.U, self.L), C.c_int32)
        self.n_h = view(s.n_h, (self.U,), C.c_int32)
        self.n_l = view(s.n_l, (self.U,), C.c_int32)
        self.req_state = view(s.req_state, (c.R,), C.c_int8)
        self.seq_len = view(s.seq_len, (c.R,), C.c_int32)
        self.pages = view(s.pages, (c.P, self.page_bytes), C.c_uint8)
        self.win_k = view(s.win_k, (self.U, c.W, c.d), C.c_uint16)
        self.win_v = view(s.win_v, (self.U, c.W, c.d), C.c_uint16)
        self.win_sig = view(s.win_sig, (self.U, c.W), C.c_float)
        self.ttable = view(s.ttable, (self.U, self.Lt), C.c_int32)      # NEXT-4 TOP table
        self.n_t = view(s.n_t, (self.U,), C.c_int32)

    def __del__(self):
        p = getattr(self, "_p", None)
        if p and _lib is not None:
            try:
                _lib.orc_pool_delete(p)
            except Exception:  # interpreter shutdown
                pass
            self._p = None

    # scalar state
    @property
    def start(self):
        return self._p.contents.start

    @start.setter
    def start(self, v):
        self._p.contents.start = v

    @property
    def free(self):
        return self._p.contents.free

    @free.setter
    def free(self, v):
        self._p.contents.free = v

    @property
    def status(self):
        return self._p.contents.status

    @property
    def last_demand(self):
        return self._p.contents.last_demand

    @property
    def last_freed(self):
        return self._p.contents.last_freed

    @property
    def oom_count(self):
        return self._p.contents.oom_count

    @property
    def last_reclaimed(self):
        return self._p.contents.last_reclaimed

    def take_status(self) -> int:
        return lib().orc_take_status(self._p)

    # calls
    def classify_decode(self, cand_sig):
        """cand_sig None: t_c's significance is taken from the window (NEXT-2)"""
        if cand_sig is not None:
            cand_sig = np.ascontiguousarray(cand_sig, dtype=np.float32)
            assert cand_sig.shape == (self.U,)
        dec = np.zeros(self.U, dtype=DECISION_DTYPE)
        st = lib().orc_classify_decode(self._p, _ptr(cand_sig), _ptr(dec))
        return st, dec

    def classify_prefill(self, req, lens, sig, want_classes=True):
        req = np.ascontiguousarray(req, dtype=np.int32)
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        sig = np.ascontiguousarray(sig, dtype=np.float32)
        n = req.shape[0]
        assert sig.shape[:2] == (n, self.LyH)
        cls = np.zeros(sig.shape, dtype=np.uint8) if want_classes else None
        st = lib().orc_classify_prefill(self._p, _ptr(req), _ptr(lens), n, _ptr(sig), sig.shape[2], _ptr(cls))
        return st, cls

    def compact_alloc(self, dec=None):
        dec = None if dec is None else np.ascontiguousarray(dec, dtype=DECISION_DTYPE)
        return lib().orc_compact_alloc(self._p, _ptr(dec))

    def quant_write_decode(self, dec, k_new, v_new, cand_sig):
        dec = np.ascontiguousarray(dec, dtype=DECISION_DTYPE)
        k_new = np.ascontiguousarray(k_new).view(np.uint16)
        v_new = np.ascontiguousarray(v_new).view(np.uint16)
        if cand_sig is not None:
            cand_sig = np.ascontiguousarray(cand_sig, dtype=np.float32)
        assert k_new.shape == (self.U, self.cfg.d)
        return lib().orc_quant_write_decode(self._p, _ptr(dec), _ptr(k_new), _ptr(v_new), _ptr(cand_sig))

    def set_head_thresholds(self, alpha_h, alpha_l):
        """NEXT-4: per-(layer, head) thresholds [Ly*H] each, or None to restore the pool-wide pair"""
        if alpha_h is None:
            return lib().orc_set_head_thresholds(self._p, None, None)
        ah = np.ascontiguousarray(alpha_h, dtype=np.float32)
        al = np.ascontiguousarray(alpha_l, dtype=np.float32)
        assert ah.shape == (self.LyH,) and al.shape == (self.LyH,)
        return lib().orc_set_head_thresholds(self._p, _ptr(ah), _ptr(al))

    def attend(self, q, want_out=True, want_probs=False):
        """NEXT-2: q = fp16 [U][G][d]; returns (status, out fp32 [U][G][d] or None, probs [U][M] or None)"""
        G = self.cfg.q_per_kv
        q = np.ascontiguousarray(q).view(np.uint16)
        assert q.shape == (self.U, G, self.cfg.d)
        out = np.zeros((self.U, G, self.cfg.d), np.float32) if want_out else None
        probs = np.zeros((self.U, self.cfg.M), np.float32) if want_probs else None
        st = lib().orc_attend(self._p, _ptr(q), _ptr(out), _ptr(probs))
        return st, out, probs

    def quant_write_prefill(self, k, v, sig):
        k = np.ascontiguousarray(k).view(np.uint16)
        v = np.ascontiguousarray(v).view(np.uint16)
        sig = np.ascontiguousarray(sig, dtype=np.float32)
        return lib().orc_quant_write_prefill(self._p, _ptr(k), _ptr(v), k.shape[2], _ptr(sig), sig.shape[2])

    def free_requests(self, req):
        req = np.ascontiguousarray(req, dtype=np.int32)
        return lib().orc_free(self._p, _ptr(req), req.shape[0])

    def prefill_conservative(self, req, lens, sig):
        req = np.ascontiguousarray(req, dtype=np.int32)
        lens = np.ascontiguousarray(lens, dtype=np.int32)
        sig = np.ascontiguousarray(sig, dtype=np.float32)
        out = np.zeros(self.cfg.P, dtype=np.int32)
        nr = C.c_int64(0)
        st = lib().orc_prefill_conservative(self._p, _ptr(req), _ptr(lens), req.shape[0], _ptr(sig), sig.shape[2],
                                            _ptr(out), C.byref(nr))
        return st, out[:nr.value].copy()

    # --- read helpers for tests (plain indexing of the documented layout) ---
    def slot_location(self, cls, u, s):
        g = self.geom[cls]
        if cls == CLS_TOP:
            return int(self.ttable[u, s // g.C]), s % g.C
        k = s // g.C if cls == CLS_HIGH else self.L - 1 - s // g.C
        return int(self.table[u, k]), s % g.C

    def slot_record(self, cls, u, s):
        """(k codes bytes, kmeta u32, v codes bytes, vmeta u32, sig bits u32, pos) of one occupied slot."""
        g = self.geom[cls]
        pid, idx = self.slot_location(cls, u, s)
        pg = self.pages[pid]
        kc = pg[g.off_k + idx * g.k_row: g.off_k + (idx + 1) * g.k_row].copy()
        vc = pg[g.off_v + idx * g.v_row: g.off_v + (idx + 1) * g.v_row].copy()
        km = int(pg[g.off_kmeta + 4 * idx: g.off_kmeta + 4 * idx + 4].view("<u4")[0]) if cls != CLS_TOP else 0
        vm = int(pg[g.off_vmeta + 4 * idx: g.off_vmeta + 4 * idx + 4].view("<u4")[0]) if cls != CLS_TOP else 0
        sg = int(pg[g.off_score + 4 * idx: g.off_score + 4 * idx + 4].view("<u4")[0])
        ps = int(pg[g.off_pos + 4 * idx: g.off_pos + 4 * idx + 4].view("<i4")[0])
        return kc, km, vc, vm, sg, ps
