"""GPU: usp_attn_fwd_host (host buffers in/out, copies inside the call).

At U = R = 1 the call pipelines H2D / attention / D2H over sequence chunks
(engine.cu fwd_host); every chunk runs the same kernel over the same key
tiles in the same order as the device-resident forward, so the results must
be BITWISE equal to usp_attn_fwd's — and the device forward is the one
tests/test_gpu_parity.py checks against the oracle. A small case is also
checked against the oracle directly. Fallback shapes (bs 2, padded head
size) must agree bitwise too.
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle
from paper_2405_07719_b200 import ProcessMesh, UspAttention
from tests.usp_harness import LSE_TOL, O_TOL, errors

pytestmark = pytest.mark.gpu


def _run(L, hc, kv, hs, causal, batch=1, seed=0):
    dev = torch.device("cuda", 0)
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs,
                       causal=causal, batch=batch, device=0)
    g = torch.Generator(device=dev).manual_seed(seed)
    # U[-1, 1) like the reference generator (the gates in usp_harness are
    # stated for that input range)
    u = lambda shape: (torch.rand(shape, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v = u(eng.q_shape()), u(eng.kv_shape()), u(eng.kv_shape())
    o, lse = eng.alloc_outputs()
    eng.forward(q, k, v, o, lse)
    torch.cuda.synchronize()
    pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)  # noqa: E731
    qh, kh, vh = pin(q), pin(k), pin(v)
    oh = torch.full(o.shape, float("nan"), dtype=o.dtype).pin_memory()
    lh = torch.full(lse.shape, float("nan"), dtype=lse.dtype).pin_memory()
    for _ in range(2):  # the second call reuses the staging buffers and chunk plans
        eng.forward_host(qh, kh, vh, oh, lh)
        torch.cuda.synchronize()
    return eng, (q, k, v), (o.cpu(), lse.cpu()), (oh, lh)


@pytest.mark.parametrize("L,hc,kv,hs,causal,batch", [
    (16384, 8, 2, 128, True, 1),    # 4 chunks of 4096 rows
    (20480, 4, 4, 64, True, 1),     # ragged last chunk
    (16384, 8, 2, 128, False, 1),   # non-causal: K/V up front, Q chunks
    (8192, 8, 2, 128, True, 2),     # bs 2: whole-tensor copies around fwd()
    (8192, 4, 2, 96, True, 1),      # padded head size: whole-tensor copies
])
def test_host_forward_bitwise_equals_device_forward(cuda, L, hc, kv, hs, causal, batch):
    eng, _, (o, lse), (oh, lh) = _run(L, hc, kv, hs, causal, batch)
    assert torch.equal(o.view(torch.int16), oh.view(torch.int16)), (o - oh).abs().max()
    assert torch.equal(lse.view(torch.int32), lh.view(torch.int32)), (lse - lh).abs().max()
    assert eng.last_launches() >= 1


def test_host_forward_matches_oracle(cuda):
    L, hc, kv, hs = 8192, 2, 1, 64
    eng, (q, k, v), _, (oh, lh) = _run(L, hc, kv, hs, True, seed=3)
    rows = np.array([0, 1, 4095, 4096, 6000, 8191])
    qd, kd, vd = (t.double().cpu().numpy() for t in (q, k, v))
    ref_o, ref_l = Oracle.softmax_rows(qd[:, rows], kd, vd, True, rows, np.arange(L))
    eo = errors(oh[:, rows].double().numpy(), ref_o)
    el = errors(lh[:, rows].double().numpy(), ref_l)
    assert eo["max_abs"] <= O_TOL and el["max_abs"] <= LSE_TOL, (eo, el)
