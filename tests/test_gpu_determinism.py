"""Repeated runs are bit-identical (no races in the persistent kernels'
dynamic unit tickets, the 2-CTA cluster ticket hand-off, the backward's
chunk hand-offs or the ring's double buffers): every unit's arithmetic is
independent of which CTA claims it. Longer runs: tools/stress.py.

The backward is bitwise repeatable in its deterministic mode
(UspAttention.set_deterministic: the two-kernel path, every dQ / dK / dV
tile summed by one CTA in a fixed order), whichever CTA runs which unit and
however many CTAs there are. The default fused backward reduces dQ
partials in arrival order: its dK / dV (and the forward) are still
bit-identical run to run, its dQ agrees to fp32 summation-order noise."""
import pytest
import torch

from paper_2405_07719_b200 import ProcessMesh, UspAttention
from tests.usp_harness import UspCase, run_usp_gpu_fwd_bwd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,hc,kv,hs", [(2048, 32, 8, 128), (2048, 8, 8, 64), (1500, 12, 4, 128)])
def test_single_rank_bitwise_repeatable(cuda, L, hc, kv, hs):
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True)
    eng.set_deterministic(True)
    g = torch.Generator(device=cuda).manual_seed(L)
    q = torch.randn(eng.q_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    k = torch.randn(eng.kv_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    v = torch.randn(eng.kv_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    do = torch.randn(eng.q_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    f0 = eng.forward(q, k, v)
    o0, l0 = f0.out.clone(), f0.logsumexp.clone()
    g0 = eng.backward(f0, do)
    ref = [g0.dq.clone(), g0.dk.clone(), g0.dv.clone()]
    for _ in range(40):
        f = eng.forward(q, k, v)
        gr = eng.backward(f, do)
        assert torch.equal(f.out, o0) and torch.equal(f.logsumexp, l0)
        assert all(torch.equal(a, b) for a, b in zip((gr.dq, gr.dk, gr.dv), ref))


def test_mesh_bitwise_repeatable(cuda):
    c = UspCase(seq=2048, hc=32, kv_hc=8, hs=128, ulysses=2, ring=4, causal=True)
    g = torch.Generator(device=cuda).manual_seed(5)
    q = torch.randn(1, c.seq, c.hc, c.hs, device=cuda, dtype=torch.bfloat16, generator=g)
    k = torch.randn(1, c.seq, c.kv_hc, c.hs, device=cuda, dtype=torch.bfloat16, generator=g)
    v = torch.randn(1, c.seq, c.kv_hc, c.hs, device=cuda, dtype=torch.bfloat16, generator=g)
    do = torch.randn(1, c.seq, c.hc, c.hs, device=cuda, dtype=torch.bfloat16, generator=g)
    ref = [x.clone() for x in run_usp_gpu_fwd_bwd(c, q, k, v, do, cuda, deterministic=True)[:4]]
    for _ in range(10):
        got = run_usp_gpu_fwd_bwd(c, q, k, v, do, cuda, deterministic=True)[:4]
        assert all(torch.equal(a, b) for a, b in zip(got, ref))


@pytest.mark.parametrize("L,hc,kv", [(2048, 32, 8), (1500, 12, 4)])
def test_fused_backward_repeatable(cuda, L, hc, kv):
    # fused backward: forward, dK and dV bit-identical; dQ within fp32
    # reduction-order noise (a few bf16 ulps at most on isolated elements)
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=128, causal=True)
    g = torch.Generator(device=cuda).manual_seed(L)
    q = torch.randn(eng.q_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    k = torch.randn(eng.kv_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    v = torch.randn(eng.kv_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    do = torch.randn(eng.q_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    f0 = eng.forward(q, k, v)
    g0 = eng.backward(f0, do)
    dq0, dk0, dv0 = g0.dq.clone(), g0.dk.clone(), g0.dv.clone()
    scale = float(dq0.float().abs().max())
    for _ in range(20):
        f = eng.forward(q, k, v)
        gr = eng.backward(f, do)
        assert torch.equal(gr.dk, dk0) and torch.equal(gr.dv, dv0)
        assert float((gr.dq.float() - dq0.float()).abs().max()) <= 1e-2 * scale


@pytest.mark.parametrize("hs", [128, 64])
def test_deterministic_dq_independent_of_grid(cuda, hs):
    """Deterministic mode: dQ / dK / dV bit-identical when the grid shrinks
    (reserved SMs change which CTA runs which unit and when)."""
    L, hc, kv = 4096, 8, 2
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True)
    eng.set_deterministic(True)
    g = torch.Generator(device=cuda).manual_seed(hs)
    q = torch.randn(eng.q_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    k = torch.randn(eng.kv_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    v = torch.randn(eng.kv_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    do = torch.randn(eng.q_shape(), device=cuda, dtype=torch.bfloat16, generator=g)
    f = eng.forward(q, k, v)
    ref = eng.backward(f, do)
    ref = [ref.dq.clone(), ref.dk.clone(), ref.dv.clone()]
    for reserve in (1, 37, 100, 140):
        eng.set_reserved_sms(reserve)
        gr = eng.backward(f, do)
        assert all(torch.equal(a, b) for a, b in zip((gr.dq, gr.dk, gr.dv), ref)), reserve
