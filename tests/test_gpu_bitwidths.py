"""GPU-vs-oracle parity for the paper's other key/value bit-width pairs (K8V8, K8V2, K4V4, K4V2 as
uniform or differentiated schemes; bits in {2, 4, 8}).  The default K8V4 / K4V2 pair has compile-time
specialisations in the bulk writer; every other pair runs its runtime-width quantizer, and the page geometry
(segment offsets, page size) changes with the widths.  Full lifecycle (prefill, decode with drift, frees,
re-admission) bit-exact after every call, then NEXT-2 attention over the same pools."""
import numpy as np
import pytest

from tests import harness as H
from tests.test_gpu_attention import _run as _run_attention
from tests.test_gpu_parity import _lifecycle

pytestmark = pytest.mark.gpu

# (high K, high V, low K, low V): K8V8 (the paper's attention-kernel experiment) over K4V4; K8V2
# over K2V2; uniform K4V2 (both classes); K8V4 over K8V2 (differentiated values only)
PAIRS = [(8, 8, 4, 4), (8, 2, 2, 2), (4, 2, 4, 2), (8, 4, 8, 2)]


@pytest.mark.parametrize("bits", PAIRS, ids=lambda b: "K%dV%d-K%dV%d" % b)
@pytest.mark.parametrize("d", [64, 128])
def test_bitwidth_lifecycle_parity(bits, d):
    kbh, vbh, kbl, vbl = bits
    scn = H.TINY.replace(R=3, Ly=2, H=3, d=d, M=600, W=32, P=5000, seed=40 + kbh + vbh + d, kbh=kbh, vbh=vbh,
                         kbl=kbl, vbl=vbl)
    _lifecycle(scn, steps=20, prompt_lens=[400, 37, 250], frees=[(6, [1])], readmit_len=170, pages_every=4)


@pytest.mark.parametrize("bits", PAIRS, ids=lambda b: "K%dV%d-K%dV%d" % b)
def test_bitwidth_attention_parity(bits):
    kbh, vbh, kbl, vbl = bits
    scn = H.TINY.replace(R=3, Ly=2, H=2, d=128, M=700, W=64, P=6000, seed=60 + kbh + vbl, q_per_kv=4,
                         kbh=kbh, vbh=vbh, kbl=kbl, vbl=vbl)
    _run_attention(scn, [520, 70, 300], steps=6, frees=[(2, [1])], readmit=150, seed=kbh)
