"""Thin ctypes binding of the C ABI in include/dkv.h (argument marshalling only).

Every function has the C name and argument order; device buffers may be passed as torch CUDA tensors or
raw integer addresses, host arrays as sequences / numpy arrays, streams as torch.cuda.Stream, raw handles
or None (= torch's current stream).  All compute runs in the sm_100a kernels of libdkv.so; there is no
fallback: importing this module raises if the library is missing, and the library returns DKV_ERR_CUDA
when no CUDA device is usable.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdkv.so")

DKV_OK, DKV_ERR_INVALID_ARG, DKV_ERR_STATE, DKV_ERR_OOM, DKV_ERR_NONFINITE, DKV_ERR_OVERFLOW, DKV_ERR_CUDA = \
    0, -1, -2, -3, -4, -5, -6
DKV_PHASE_DECODE, DKV_PHASE_PREFILL = 0, 1
DKV_CLS_NONE, DKV_CLS_HIGH, DKV_CLS_LOW, DKV_CLS_PRUNED = 0, 1, 2, 3
DKV_V_NONE, DKV_V_KEEP, DKV_V_DOWN, DKV_V_PRUNE = 0, 1, 2, 3
DKV_GROW_NONE, DKV_GROW_HIGH, DKV_GROW_LOW = 0, 1, 2
DKV_REQ_IDLE, DKV_REQ_ADMITTING, DKV_REQ_ACTIVE, DKV_REQ_PENDING_FREE = 0, 1, 2, 3

EXPORTED = ("dkv_arena_bytes", "dkv_pool_layout", "dkv_pool_init", "dkv_pool_destroy", "dkv_classify",
            "dkv_compact_alloc", "dkv_quant_write", "dkv_free", "dkv_pool_query", "dkv_pool_stats_device_ptr",
            "dkv_status_string", "dkv_attend", "dkv_set_head_thresholds", "dkv_decode_stage_bytes",
            "dkv_decode_step_host", "dkv_decode_graph_create", "dkv_decode_graph_launch",
            "dkv_decode_graph_kernel_ms", "dkv_decode_graph_destroy", "dkv_attend_tc", "dkv_audit")


class DkvError(RuntimeError):
    def __init__(self, fn, status):
        self.status = status
        super().__init__(f"{fn} failed: {status} ({status_string(status)})")


class dkv_config_t(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "max_requests", "num_layers", "num_kv_heads", "head_dim", "max_seq_len", "window", "page_tokens_high",
        "page_tokens_low", "kbits_high", "vbits_high", "kbits_low", "vbits_low", "num_pages")] + \
        [("alpha_h", C.c_float), ("alpha_l", C.c_float), ("prompt_denominator", C.c_int32),
         ("tile_units", C.c_int32), ("prefill_workflow", C.c_int32), ("q_per_kv", C.c_int32),
         ("top_tier", C.c_int32), ("alpha_t", C.c_float), ("page_tokens_top", C.c_int32)]


class dkv_decision_t(C.Structure):
    _fields_ = [("tc_class", C.c_uint8), ("v_action", C.c_uint8), ("grow", C.c_uint8), ("demand", C.c_uint8),
                ("v_slot", C.c_int32), ("tc_slot", C.c_int32), ("v_dst_slot", C.c_int32)]


class dkv_stats_t(C.Structure):
    _fields_ = [("free_pages", C.c_int64), ("used_pages", C.c_int64), ("start", C.c_int64),
                ("last_demand", C.c_int64), ("last_freed", C.c_int64), ("status", C.c_int32),
                ("oom_count", C.c_int32)]


class dkv_layout_t(C.Structure):
    _fields_ = [("arena_bytes", C.c_int64)] + [(n, C.c_int64) for n in (
        "off_ctrl", "off_tile_status", "off_ring", "off_table", "off_n_h", "off_n_l", "off_req_state",
        "off_seq_len", "off_prompt_len", "off_admit", "off_pf_nh", "off_pf_nl", "off_pf_seg", "off_win_k",
        "off_win_v", "off_pages", "off_stats")] + [(n, C.c_int32) for n in (
        "units", "table_len", "page_bytes", "num_tiles", "tile_units", "seg_tokens", "num_segs")] + \
        [(n, C.c_int32 * 3) for n in ("C", "k_row", "v_row", "off_k", "off_kmeta", "off_v", "off_vmeta",
                                       "off_score", "off_pos")] + [("off_tile_sums", C.c_int64), ("off_rec", C.c_int64),
                                                                  ("off_win_sig", C.c_int64), ("off_secmin", C.c_int64),
                                                                  ("off_head_alpha", C.c_int64),
                                                                  ("off_att_scratch", C.c_int64),
                                                                  ("off_ttable", C.c_int64), ("off_n_t", C.c_int64),
                                                                  ("table_len_top", C.c_int32), ("C_top", C.c_int32),
                                                                  ("row_top", C.c_int32), ("off_k_top", C.c_int32),
                                                                  ("off_v_top", C.c_int32), ("off_score_top", C.c_int32),
                                                                  ("off_pos_top", C.c_int32), ("off_qpid", C.c_int64),
                                                                  ("off_tsum", C.c_int64),
                                                                  ("off_tc_scratch", C.c_int64)]


assert C.sizeof(dkv_decision_t) == 16

DECISION_DTYPE = np.dtype([("tc_class", "u1"), ("v_action", "u1"), ("grow", "u1"), ("demand", "u1"),
                           ("v_slot", "<i4"), ("tc_slot", "<i4"), ("v_dst_slot", "<i4")])

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing — build it first (python -c 'import __graft_entry__ as g; g.build()')")

_lib = C.CDLL(LIB_PATH)
_P = C.POINTER
_vp = C.c_void_p
_lib.dkv_arena_bytes.argtypes = [_P(dkv_config_t)]
_lib.dkv_arena_bytes.restype = C.c_size_t
_lib.dkv_pool_layout.argtypes = [_P(dkv_config_t), _P(dkv_layout_t)]
_lib.dkv_pool_init.argtypes = [_P(dkv_config_t), _vp, C.c_size_t, _vp, _P(_vp)]
_lib.dkv_pool_destroy.argtypes = [_vp]
_lib.dkv_classify.argtypes = [_vp, C.c_int32, _vp, _vp, C.c_int32, _vp, C.c_int64, _vp, _vp, _vp]
_lib.dkv_compact_alloc.argtypes = [_vp, _vp, _vp]
_lib.dkv_quant_write.argtypes = [_vp, C.c_int32, _vp, _vp, _vp, C.c_int64, _vp, C.c_int64, _vp]
_lib.dkv_free.argtypes = [_vp, _vp, C.c_int32, _vp]
_lib.dkv_attend.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.dkv_attend_tc.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.dkv_audit.argtypes = [_vp, _vp, _vp, _vp]
_lib.dkv_set_head_thresholds.argtypes = [_vp, _vp, _vp, _vp]
_lib.dkv_pool_query.argtypes = [_vp, _P(dkv_stats_t), _vp]
_lib.dkv_decode_stage_bytes.argtypes = [_vp]
_lib.dkv_decode_stage_bytes.restype = C.c_size_t
_lib.dkv_decode_step_host.argtypes = [_vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]
_lib.dkv_pool_stats_device_ptr.argtypes = [_vp]
_lib.dkv_pool_stats_device_ptr.restype = _vp
_lib.dkv_decode_graph_create.argtypes = [_vp, C.c_int32, _vp, C.c_int64, _vp, _vp, C.c_int64, _vp, C.c_int32, _P(_vp)]
_lib.dkv_decode_graph_launch.argtypes = [_vp, _vp]
_lib.dkv_decode_graph_kernel_ms.argtypes = [_vp, _vp]
_lib.dkv_decode_graph_destroy.argtypes = [_vp]
_lib.dkv_status_string.argtypes = [C.c_int32]
_lib.dkv_status_string.restype = C.c_char_p
for _f in ("dkv_pool_layout", "dkv_pool_init", "dkv_pool_destroy", "dkv_classify", "dkv_compact_alloc",
           "dkv_quant_write", "dkv_free", "dkv_pool_query", "dkv_attend", "dkv_set_head_thresholds",
           "dkv_decode_step_host", "dkv_decode_graph_create", "dkv_decode_graph_launch", "dkv_decode_graph_kernel_ms",
           "dkv_decode_graph_destroy", "dkv_attend_tc", "dkv_audit"):
    getattr(_lib, _f).restype = C.c_int32


def lib():
    return _lib


# ------------------------------------------------------------------------------------------ marshalling
def _dev(x):
    """Device address of a torch tensor / integer / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_cuda:
            raise ValueError("expected a CUDA tensor for a device buffer")
        if not x.is_contiguous():
            raise ValueError("device buffers must be contiguous")
        return x.data_ptr()
    raise TypeError(f"cannot pass {type(x)} as a device buffer")


def _stream(s):
    if s is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _host_i32(a):
    if a is None:
        return None, None
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return arr, arr.ctypes.data_as(_vp)


def status_string(st: int) -> str:
    return _lib.dkv_status_string(int(st)).decode()


def _check(fn, st):
    if st != DKV_OK:
        raise DkvError(fn, st)
    return st


# ------------------------------------------------------------------------------------------ C names
def dkv_arena_bytes(cfg: dkv_config_t) -> int:
    return int(_lib.dkv_arena_bytes(C.byref(cfg)))


def dkv_pool_layout(cfg: dkv_config_t) -> dkv_layout_t:
    out = dkv_layout_t()
    _check("dkv_pool_layout", _lib.dkv_pool_layout(C.byref(cfg), C.byref(out)))
    return out


def dkv_pool_init(cfg: dkv_config_t, d_arena, arena_bytes: int, stream=None) -> int:
    h = _vp()
    _check("dkv_pool_init", _lib.dkv_pool_init(C.byref(cfg), _dev(d_arena), arena_bytes, _stream(stream), C.byref(h)))
    return h.value


def dkv_pool_destroy(pool: int) -> int:
    return _check("dkv_pool_destroy", _lib.dkv_pool_destroy(pool))


def dkv_classify(pool, phase, h_req, h_len, n, d_sig, sig_stride, d_dec, d_token_class, stream=None) -> int:
    req, preq = _host_i32(h_req)
    ln, pln = _host_i32(h_len)
    return _check("dkv_classify", _lib.dkv_classify(pool, phase, preq, pln, n, _dev(d_sig), sig_stride, _dev(d_dec),
                                                    _dev(d_token_class), _stream(stream)))


def dkv_compact_alloc(pool, d_dec, stream=None) -> int:
    return _check("dkv_compact_alloc", _lib.dkv_compact_alloc(pool, _dev(d_dec), _stream(stream)))


def dkv_quant_write(pool, phase, d_dec, d_k, d_v, kv_stride, d_sig, sig_stride, stream=None) -> int:
    return _check("dkv_quant_write", _lib.dkv_quant_write(pool, phase, _dev(d_dec), _dev(d_k), _dev(d_v), kv_stride,
                                                          _dev(d_sig), sig_stride, _stream(stream)))


def dkv_attend(pool, d_q, d_out, d_probs, stream=None) -> int:
    return _check("dkv_attend", _lib.dkv_attend(pool, _dev(d_q), _dev(d_out), _dev(d_probs), _stream(stream)))


def dkv_attend_tc(pool, d_q, d_out, d_probs, stream=None) -> int:
    return _check("dkv_attend_tc", _lib.dkv_attend_tc(pool, _dev(d_q), _dev(d_out), _dev(d_probs), _stream(stream)))


def dkv_audit(pool, d_scratch, d_result, stream=None) -> int:
    return _check("dkv_audit", _lib.dkv_audit(pool, _dev(d_scratch), _dev(d_result), _stream(stream)))


def dkv_set_head_thresholds(pool, alpha_h, alpha_l, stream=None) -> int:
    if alpha_h is None:
        return _check("dkv_set_head_thresholds", _lib.dkv_set_head_thresholds(pool, None, None, _stream(stream)))
    ah = np.ascontiguousarray(np.asarray(alpha_h, dtype=np.float32))
    al = np.ascontiguousarray(np.asarray(alpha_l, dtype=np.float32))
    return _check("dkv_set_head_thresholds", _lib.dkv_set_head_thresholds(
        pool, ah.ctypes.data_as(_vp), al.ctypes.data_as(_vp), _stream(stream)))


def dkv_decode_stage_bytes(pool) -> int:
    return int(_lib.dkv_decode_stage_bytes(pool))


def _hostp(x):
    """Host address of a CPU torch tensor / numpy array / None (pinned CPU tensors give asynchronous copies)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        if x.is_cuda or not x.is_contiguous():
            raise ValueError("expected a contiguous host (CPU) tensor")
        return x.data_ptr()
    if not x.flags["C_CONTIGUOUS"]:
        raise ValueError("expected a C-contiguous host array")
    return x.ctypes.data


def dkv_decode_step_host(pool, h_sig, h_kv, h_dec, d_stage, stage_bytes, stream=None) -> int:
    return _check("dkv_decode_step_host", _lib.dkv_decode_step_host(pool, _hostp(h_sig), _hostp(h_kv), _hostp(h_dec),
                                                                    _dev(d_stage), stage_bytes, _stream(stream)))


DKV_GRAPH_PDL, DKV_GRAPH_EVENTS = 1, 2


def dkv_decode_graph_create(pool, steps, d_sig, sig_step, d_k, d_v, kv_step, d_dec, flags) -> int:
    h = _vp()
    _check("dkv_decode_graph_create", _lib.dkv_decode_graph_create(pool, steps, _dev(d_sig), sig_step, _dev(d_k),
                                                                   _dev(d_v), kv_step, _dev(d_dec), flags, C.byref(h)))
    return h.value


def dkv_decode_graph_launch(graph, stream=None) -> int:
    return _check("dkv_decode_graph_launch", _lib.dkv_decode_graph_launch(graph, _stream(stream)))


def dkv_decode_graph_kernel_ms(graph, steps) -> np.ndarray:
    out = np.zeros((steps, 3), np.float32)
    _check("dkv_decode_graph_kernel_ms", _lib.dkv_decode_graph_kernel_ms(graph, out.ctypes.data_as(_vp)))
    return out


def dkv_decode_graph_destroy(graph) -> int:
    return _check("dkv_decode_graph_destroy", _lib.dkv_decode_graph_destroy(graph))


def dkv_free(pool, h_req, n, stream=None) -> int:
    req, preq = _host_i32(h_req)
    return _check("dkv_free", _lib.dkv_free(pool, preq, n, _stream(stream)))


def dkv_pool_query(pool, stream=None):
    """Returns (device status, dkv_stats_t); the device status is returned, not raised."""
    out = dkv_stats_t()
    st = _lib.dkv_pool_query(pool, C.byref(out), _stream(stream))
    if st == DKV_ERR_CUDA or st == DKV_ERR_INVALID_ARG:
        raise DkvError("dkv_pool_query", st)
    return st, out


def dkv_pool_stats_device_ptr(pool) -> int:
    return int(_lib.dkv_pool_stats_device_ptr(pool))


def dkv_status_string(st) -> str:
    return status_string(st)


def make_config(R, Ly, H, d, M, W, Ch=16, Cl=32, kbh=8, vbh=4, kbl=4, vbl=2, P=1024, alpha_h=1.0, alpha_l=0.02,
                prompt_denominator=0, tile_units=0, prefill_workflow=0, q_per_kv=0, top_tier=0, alpha_t=0.0,
                page_tokens_top=4) -> dkv_config_t:
    c = dkv_config_t(max_requests=R, num_layers=Ly, num_kv_heads=H, head_dim=d, max_seq_len=M, window=W,
                     page_tokens_high=Ch, page_tokens_low=Cl, kbits_high=kbh, vbits_high=vbh, kbits_low=kbl,
                     vbits_low=vbl, num_pages=P, alpha_h=alpha_h, alpha_l=alpha_l,
                     prompt_denominator=prompt_denominator, tile_units=tile_units,
                     prefill_workflow=prefill_workflow, q_per_kv=q_per_kv, top_tier=top_tier, alpha_t=alpha_t,
                     page_tokens_top=page_tokens_top)
    return c
