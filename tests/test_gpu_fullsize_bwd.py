"""Backward parity at full sizes (SURVEY §8(f) #1 at BASELINE.json's lengths).

The small-L backward tests (tests/test_gpu_backward.py) compare whole
gradients with the oracle's usp_attention_backward restatement; at 32K-128K
that is hours of fp64 CPU work, so here the engine runs the WHOLE
configuration and a seeded sample of gradient rows is recomputed in fp64
from the definitions the oracle restates (attention.cpp:266-324):

    P[q,k]  = exp(S[q,k] / sqrt(hs) - lse[q])        (causal: k <= q)
    dP[q,k] = dO[q] . V[k],   delta[q] = dO[q] . O[q]
    dS      = P (dP - delta) / sqrt(hs)
    dQ[q]   = sum_k dS[q,k] K[k]
    dK[k]   = sum_{q, heads of k's group} dS[q,k] Q[q]
    dV[k]   = sum_{q, heads of k's group} P[q,k] dO[q]

taking the forward's O and LSE from the GPU (checked against the oracle at
these sizes by tests/test_gpu_fullsize.py). Both backward algorithms run:
the fused kernel (default) and the deterministic two-kernel path.

Tolerance: as tests/test_gpu_backward.py, over the sampled rows: relative L2
<= 2e-2 and max-abs <= 2e-2 * max|ref| per gradient.
"""
import numpy as np
import pytest
import torch

from paper_2405_07719_b200 import ProcessMesh, UspAttention

pytestmark = pytest.mark.gpu
K = 1024
REL_L2 = 2e-2
MAX_REL = 2e-2


def _sampled_grads(q, k, v, o, lse, do, qrows, krows):
    """fp64 dQ rows `qrows` and dK/dV rows `krows` (causal, positions = row index)."""
    L, hc, hs = q.shape[1], q.shape[2], q.shape[3]
    kv = k.shape[2]
    g = hc // kv
    sc = 1.0 / np.sqrt(hs)
    Q, Kt, V = (x[0].double().cpu().numpy() for x in (q, k, v))
    O, dO = o[0].double().cpu().numpy(), do[0].double().cpu().numpy()
    LSE = lse[0].double().cpu().numpy()  # (L, hc), natural log
    delta = np.einsum("lhd,lhd->lh", dO, O)
    dq = np.zeros((len(qrows), hc, hs))
    for i, r in enumerate(qrows):
        for h in range(hc):
            kh = h // g
            s = Kt[: r + 1, kh] @ Q[r, h] * sc
            p = np.exp(s - LSE[r, h])
            dp = V[: r + 1, kh] @ dO[r, h]
            ds = p * (dp - delta[r, h]) * sc
            dq[i, h] = ds @ Kt[: r + 1, kh]
    dk = np.zeros((len(krows), kv, hs))
    dv = np.zeros((len(krows), kv, hs))
    for i, c in enumerate(krows):
        for kh in range(kv):
            for h in range(kh * g, (kh + 1) * g):
                s = Q[c:, h] @ Kt[c, kh] * sc
                p = np.exp(s - LSE[c:, h])
                dp = dO[c:, h] @ V[c, kh]
                ds = p * (dp - delta[c:, h]) * sc
                dv[i, kh] += p @ dO[c:, h]
                dk[i, kh] += ds @ Q[c:, h]
    return dq, dk, dv


def _check(name, got, want):
    d = got - want
    rel = float(np.linalg.norm(d) / np.linalg.norm(want))
    mx = float(np.abs(d).max())
    scale = float(np.abs(want).max())
    assert np.isfinite(got).all(), name
    assert rel <= REL_L2 and mx <= MAX_REL * scale, (name, rel, mx, scale)
    return rel


@pytest.mark.parametrize("L,det", [(32 * K, False), (32 * K, True), (128 * K, False)])
def test_full_size_backward_sampled_rows(cuda, L, det):
    hc, kv, hs = 32, 8, 128
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True)
    eng.set_deterministic(det)
    gen = torch.Generator(device=cuda).manual_seed(L + det)
    u = lambda *s: (torch.rand(s, device=cuda, generator=gen) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v, do = u(1, L, hc, hs), u(1, L, kv, hs), u(1, L, kv, hs), u(1, L, hc, hs)
    fwd = eng.forward(q, k, v)
    grads = eng.backward(fwd, do)
    torch.cuda.synchronize()
    rng = np.random.default_rng(L)
    # first / last rows, tile edges, random rows
    nr = 10 if L <= 32 * K else 3  # the fp64 rows cost O(L) each
    qrows = np.unique(np.concatenate([[0, 1, 127, 128, L - 129, L - 1], rng.integers(0, L, nr)]))
    krows = np.unique(np.concatenate([[0, 127, 128, L - 128, L - 1], rng.integers(0, L, nr)]))
    dq, dk, dv = _sampled_grads(q, k, v, fwd.out, fwd.logsumexp, do, qrows, krows)
    rels = [
        _check("dq", grads.dq[0, qrows].double().cpu().numpy(), dq),
        _check("dk", grads.dk[0, krows].double().cpu().numpy(), dk),
        _check("dv", grads.dv[0, krows].double().cpu().numpy(), dv),
    ]
    print(f"L={L} det={det}: rel L2 dQ/dK/dV = {rels}")
    assert eng.last_launches() >= (5 if not det else 6)
    eng.close()
