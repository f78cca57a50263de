"""GPU parity of the backward: usp_attn_bwd through the C
ABI vs the oracle's restatement of usp_attention_backward (usp_attention.cpp:
68-89, ring_attention.cpp:79-155, attention.cpp:266-324), itself pinned
bitwise to the reference (tests/test_oracle.py::test_backward_*).

Inputs: Q, K, V, dO from one UniformSource stream (usp_harness.hpp:30-41)
rounded to bf16; the oracle runs in fp64 on the same bf16 values widened.

Tolerance (bf16 operands incl. P and dS, fp32 accumulation, vs fp64):
  per gradient, relative L2 <= 2e-2 and max-abs <= 2e-2 * max|ref|.

Both backward algorithms run every case: the fused kernel (default at head
size 128: one kernel per ring step, dQ reduced with fp32 atomics) and the
deterministic two-kernel path (`det` parameter). The launch count tells
which ran: per ring step the fused path launches one attention kernel (+ the
partial's add at t >= 2), the two-kernel path two.
"""
import numpy as np
import pytest

from oracle.oracle import oracle_reference_attention_grad, oracle_usp_backward
from tests.usp_harness import UspCase, errors, make_globals_with_dout, run_usp_gpu_fwd_bwd, to_bf16, widen

REL_L2 = 2e-2
MAX_REL = 2e-2

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[False, True], ids=["fused", "det"])
def det(request):
    return request.param


def _expected_launches(c: UspCase, det: bool) -> int:
    """Kernels of one usp_attn_bwd on a rank: pack + unpack of dO when U > 1
    is counted by the engine too, so only the attention part is asserted:
    delta (1), per ring step one fused kernel (+1 add at t >= 2) or two."""
    R = c.ring
    fused = not det
    return 1 + (R + max(0, R - 2) if fused else 2 * R)


def _check(c: UspCase, device, det: bool = False):
    q, k, v, do = make_globals_with_dout(c)
    tq, tk, tv, tdo = (to_bf16(x, device) for x in (q, k, v, do))
    _, dq, dk, dv, engines, _ = run_usp_gpu_fwd_bwd(c, tq, tk, tv, tdo, device, deterministic=det)
    args = [widen(x) for x in (tq, tk, tv, tdo)]
    if c.ulysses * c.ring == 1:
        ref = oracle_reference_attention_grad(*args, c.causal)
    else:
        ref = oracle_usp_backward(*args, c.ulysses, c.ring, c.causal)
    res = {}
    for name, got, want in zip(("dq", "dk", "dv"), (dq, dk, dv), ref):
        g = widen(got)
        e = errors(g, want)
        res[name] = e
        scale = float(np.abs(want).max())
        assert np.isfinite(g).all(), (c, name)
        assert e["rel_l2"] <= REL_L2 and e["max_abs"] <= MAX_REL * scale, (c, name, e, scale)
    # the attention kernels of the selected algorithm ran (the rest is
    # reshard / cast work: at least the three casts)
    want = _expected_launches(c, det) + 3
    assert all(e.last_launches() >= want for e in engines), ("backward kernels", [e.last_launches() for e in engines], want)
    return res


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("shape", [(512, 8, 2, 128), (640, 4, 4, 64), (1000, 4, 1, 128), (384, 6, 3, 128)])
def test_single_rank_backward(cuda, shape, causal, det):
    L, hc, kv, hs = shape
    _check(UspCase(seq=L, hc=hc, kv_hc=kv, hs=hs, causal=causal, seed=17 + L), cuda, det)


def test_single_rank_backward_batch2_padded_head_size(cuda):
    _check(UspCase(bs=2, seq=256, hc=4, kv_hc=2, hs=4, causal=True, seed=91), cuda)
    _check(UspCase(bs=1, seq=300, hc=2, kv_hc=1, hs=96, causal=False, seed=92), cuda)


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("u,r", [(1, 8), (2, 4), (4, 2), (8, 1)])
def test_backward_factorizations_of_8(cuda, u, r, causal, det):
    # test_usp.cpp's factorization sweep applied to the backward.
    _check(UspCase(seq=2048, hc=8, kv_hc=8, hs=128, ulysses=u, ring=r, causal=causal, seed=4242), cuda, det)


@pytest.mark.parametrize("u,r", [(1, 8), (2, 4), (4, 2), (8, 1)])
def test_backward_reference_tiny(cuda, u, r):
    for causal in (True, False):
        _check(UspCase(seq=32, hc=8, kv_hc=8, hs=4, ulysses=u, ring=r, causal=causal, seed=4242), cuda)


def test_backward_gqa_hybrid_batch2(cuda, det):
    _check(UspCase(bs=2, seq=512, hc=8, kv_hc=2, hs=128, ulysses=2, ring=2, causal=True, seed=999), cuda, det)


def test_backward_ring3_llama_heads(cuda, det):
    _check(UspCase(seq=1536, hc=32, kv_hc=8, hs=128, ulysses=2, ring=3, causal=True, seed=3), cuda, det)


@pytest.mark.parametrize("u,r", [(1, 4), (2, 4)])
def test_backward_fused_ring_partials(cuda, u, r):
    # R >= 3 exercises the fused path's scratch block + add into the
    # circulating partial (t >= 2); GQA group 4 with q-head-innermost tiles
    _check(UspCase(seq=4096, hc=32, kv_hc=8, hs=128, ulysses=u, ring=r, causal=True, seed=77), cuda, False)


def test_backward_ledger_matches_plan(cuda):
    from paper_2405_07719_b200.usp import backward_ledger

    c = UspCase(seq=1536, hc=8, kv_hc=4, hs=128, ulysses=2, ring=3, causal=True, seed=5)
    q, k, v, do = make_globals_with_dout(c)
    tq, tk, tv, tdo = (to_bf16(x, cuda) for x in (q, k, v, do))
    for det in (False, True):
        _, _, _, _, engines, _ = run_usp_gpu_fwd_bwd(c, tq, tk, tv, tdo, cuda, deterministic=det)
        for e in engines:
            assert e.ledger() == backward_ledger(e.cfg), (e.rank, det)


def test_backward_without_forward_is_rejected(cuda):
    import torch

    from paper_2405_07719_b200 import ProcessMesh, UspAttention, UspForward, UspInvalidInput
    from paper_2405_07719_b200._lib import check, lib
    from paper_2405_07719_b200.usp import _ptr

    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=256, heads=4, kv_heads=2, head_size=128, causal=True)
    q = torch.zeros(eng.q_shape(), dtype=torch.bfloat16, device=cuda)
    kv = torch.zeros(eng.kv_shape(), dtype=torch.bfloat16, device=cuda)
    lse = torch.zeros(eng.lse_shape(), dtype=torch.float32, device=cuda)
    with pytest.raises(UspInvalidInput, match="missing forward artifacts"):
        check(lib().usp_attn_bwd(eng._h, _ptr(q), _ptr(kv), _ptr(kv), _ptr(q), _ptr(lse), _ptr(q), _ptr(q),
                                 _ptr(kv), _ptr(kv), None))
    with pytest.raises(UspInvalidInput, match="missing forward artifacts"):
        eng.backward(UspForward(q, lse, []), q)
    eng.close()
