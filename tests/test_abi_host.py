"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol include/dkv.h
declares, its arena layout agrees with the oracle's independent geometry, invalid configurations are
rejected, and without a device every entry point fails loudly (DKV_ERR_CUDA) — there is no CPU path."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def D():
    so = os.path.join(ROOT, "paper_2412_03131_b200", "libdkv.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-C", ROOT, "-j8"])
    from paper_2412_03131_b200 import dkv
    return dkv


def test_exports_every_header_symbol(D):
    hdr = open(os.path.join(ROOT, "include", "dkv.h")).read()
    names = set(re.findall(r"^\s*(?:size_t|dkv_status_t|int64_t\*|const char\*)\s+(dkv_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 11
    lib = C.CDLL(D.LIB_PATH)
    for n in sorted(names):
        assert hasattr(lib, n), f"libdkv.so does not export {n}"
    assert names == set(D.EXPORTED)


def test_layout_matches_oracle_geometry(D):
    import oracle
    for kw in (dict(R=4, Ly=2, H=4, d=64, M=128, W=16, Ch=16, Cl=32, P=1024),
               dict(R=64, Ly=32, H=8, d=128, M=8192, W=64, Ch=16, Cl=32, P=1 << 22),
               dict(R=3, Ly=1, H=5, d=128, M=300, W=4, Ch=8, Cl=8, kbh=4, vbh=2, kbl=2, vbl=2, P=77),
               dict(R=32, Ly=64, H=2, d=128, M=33792, W=64, Ch=16, Cl=32, P=1000)):
        cfg = D.make_config(kw["R"], kw["Ly"], kw["H"], kw["d"], kw["M"], kw["W"], kw["Ch"], kw["Cl"],
                            kw.get("kbh", 8), kw.get("vbh", 4), kw.get("kbl", 4), kw.get("vbl", 2), kw["P"])
        lay = D.dkv_pool_layout(cfg)
        geo = oracle.geometry(oracle.make_config(**kw))
        assert (lay.units, lay.table_len, lay.page_bytes) == (geo["U"], geo["L"], geo["page_bytes"])
        for c, g in ((1, geo["high"]), (2, geo["low"])):
            for f in ("C", "k_row", "v_row", "off_k", "off_kmeta", "off_v", "off_vmeta", "off_score", "off_pos"):
                assert getattr(lay, f)[c] == getattr(g, f), (kw, c, f)
        assert lay.arena_bytes >= kw["P"] * lay.page_bytes
        assert lay.off_pages % 4096 == 0


def test_llama8b_layout_figures(D):
    # U = 16384, L = 512, page = 3584 B; high 16 tokens K8V4 = 3328 used bytes, low 32 K4V2
    lay = D.dkv_pool_layout(D.make_config(64, 32, 8, 128, 8192, 64, 16, 32, P=1 << 22))
    assert (lay.units, lay.table_len, lay.page_bytes) == (16384, 512, 3584)
    assert list(lay.off_score)[1:] == [3200, 3328] and list(lay.off_pos)[1:] == [3264, 3456]


@pytest.mark.parametrize("bad", [dict(d=96), dict(Ch=6), dict(Cl=8, Ch=16), dict(kbh=3), dict(P=0), dict(W=-1),
                                 dict(alpha_h=float("nan")), dict(alpha_l=-1.0), dict(M=0), dict(tile_units=300)])
def test_invalid_configs_rejected(D, bad):
    kw = dict(R=4, Ly=2, H=4, d=64, M=128, W=16, Ch=16, Cl=32, P=1024)
    kw.update(bad)
    cfg = D.make_config(kw["R"], kw["Ly"], kw["H"], kw["d"], kw["M"], kw["W"], kw["Ch"], kw["Cl"],
                        kw.get("kbh", 8), 4, 4, 2, kw["P"], kw.get("alpha_h", 1.0), kw.get("alpha_l", 0.02), 0,
                        kw.get("tile_units", 0))
    assert D.dkv_arena_bytes(cfg) == 0
    with pytest.raises(D.DkvError) as e:
        D.dkv_pool_layout(cfg)
    assert e.value.status == D.DKV_ERR_INVALID_ARG


def test_no_device_fails_loudly(D):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    cfg = D.make_config(4, 2, 4, 64, 128, 16)
    n = D.dkv_arena_bytes(cfg)
    h = C.c_void_p()
    st = D.lib().dkv_pool_init(C.byref(cfg), C.c_void_p(1 << 20), n, None, C.byref(h))
    assert st == D.DKV_ERR_CUDA and not h.value
    assert D.lib().dkv_classify(None, 0, None, None, 0, None, 0, None, None, None) == D.DKV_ERR_INVALID_ARG
    # the host-buffer decode step validates its arguments before any CUDA call
    assert D.lib().dkv_decode_stage_bytes(None) == 0
    buf = (C.c_uint16 * 8)()
    assert D.lib().dkv_decode_step_host(None, None, buf, None, C.c_void_p(1 << 20), 1 << 20, None) == D.DKV_ERR_INVALID_ARG
    # the decode-graph calls reject a NULL handle / output without touching CUDA
    g = C.c_void_p()
    assert D.lib().dkv_decode_graph_create(None, 1, None, 0, buf, buf, 0, buf, 0, C.byref(g)) == D.DKV_ERR_INVALID_ARG
    assert not g.value
    assert D.lib().dkv_decode_graph_launch(None, None) == D.DKV_ERR_INVALID_ARG
    assert D.lib().dkv_decode_graph_kernel_ms(None, buf) == D.DKV_ERR_INVALID_ARG
    assert D.lib().dkv_decode_graph_destroy(None) == D.DKV_ERR_INVALID_ARG


def test_status_strings(D):
    for st in (0, -1, -2, -3, -4, -5, -6):
        assert D.status_string(st) and D.status_string(st) != "unknown status"
