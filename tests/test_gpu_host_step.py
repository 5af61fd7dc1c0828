"""GPU-vs-oracle parity of dkv_decode_step_host — the whole decode step from HOST buffers (the e2e path of
bench.py; include/dkv.h): the significance and the new tokens' K/V copied in by the library (K/V on its own
copy stream), classify -> compact_alloc -> quant_write, the decisions copied back.  The oracle runs the
same step as three calls; decisions and the whole pool state must be bit-identical after every step, across
a free (recycling step) and a re-admission."""
import numpy as np
import pytest
import torch

from tests import harness as H

pytestmark = pytest.mark.gpu


def _host_step(o, g, inp, life, step):
    from tests.gpu_backend import compare_state, dec_np
    o.drift(step)
    g.drift(step)
    active = life.state == H.REQ_ACTIVE
    N = np.where(active, life.seq + 1, 0)
    cand, k, v = inp.decode(N)
    st, dec_o = o.classify_decode(cand)
    assert st == 0
    assert o.compact_alloc(dec_o) == 0
    assert o.quant_write_decode(dec_o, k, v, cand) == 0
    h_sig = torch.as_tensor(np.asarray(cand, np.float32)).contiguous().pin_memory()
    kk = torch.as_tensor(k).view(torch.int16) if isinstance(k, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(k).view(np.int16))
    vv = torch.as_tensor(v).view(torch.int16) if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v).view(np.int16))
    h_kv = torch.stack([kk.reshape(g.U, -1), vv.reshape(g.U, -1)]).contiguous().pin_memory()
    h_dec = torch.full((g.U, 4), -7, dtype=torch.int32).pin_memory()
    g.pool.decode_step_host(h_sig, h_kv, h_dec)
    torch.cuda.synchronize()
    a = dec_np(dec_o)
    b = h_dec.numpy()
    assert np.array_equal(np.ascontiguousarray(a).view(np.uint8).reshape(-1), b.view(np.uint8).reshape(-1)), \
        f"host-step decisions differ at step {step}"
    compare_state(o.snapshot(), g.snapshot(), where=f"host step {step}")
    life.seq[active] += 1


@pytest.mark.parametrize("tile_units", [0, 256])
def test_decode_step_host_matches_oracle(tile_units):
    from tests.gpu_backend import GpuBackend, compare_state
    # the tiny config (BASELINE configs[0]) and a multi-tile ragged pool (3 x 256-unit tiles, 600 units)
    scn = H.TINY if tile_units == 0 else H.Scenario(R=8, Ly=3, H=25, M=160, P=8192, tile_units=tile_units)
    lens = [64] * scn.R if tile_units == 0 else [40, 90, 17, 128, 64, 33, 100, 75]
    o, g = H.OracleBackend(scn), GpuBackend(scn)
    inp, life = H.Inputs(scn), H.Lifecycle(scn)
    H.admit([o, g], inp, life, list(range(scn.R)), lens)
    compare_state(o.snapshot(), g.snapshot(), where="admit")
    for step in range(12):
        _host_step(o, g, inp, life, step)
        if step == 4:
            H.free([o, g], life, [1])
        if step == 6:
            assert o.pool.req_state[1] == 0
            H.admit([o, g], inp, life, [1], [48])
            compare_state(o.snapshot(), g.snapshot(), where="re-admit")
