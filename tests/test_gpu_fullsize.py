"""GPU parity at BASELINE.json's full sizes (the
sampled-row oracle).

A full fp64 oracle at L = 128K-208K takes hours on the CPU, so each case runs
the engine on the WHOLE configuration (every rank of the U x R mesh through
the in-process transport on one GPU, zigzag layout) and checks a seeded
sample of query rows — the first and last rows, the zigzag chunk edges and
random rows — against the oracle's SoftmaxState restatement of those rows
over ALL keys (oracle.softmax_rows, pinned bitwise to the reference in
tests/test_oracle.py). O is compared in original token order after
place_rows; LSE in the head-sharded layout of the rank that owns each row.

Inputs: uniform [-1, 1) from a seeded torch generator on the GPU, rounded to
bf16 (the reference generator's host stream would need 4-8 GB of fp64 here);
the oracle runs on the same bf16 values widened to fp64.
Tolerance: as tests/test_gpu_parity.py (O max-abs 5e-3, LSE max-abs 1e-4).
"""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle
from tests.usp_harness import LSE_TOL, O_TOL, UspCase, errors, run_usp_gpu, widen

pytestmark = pytest.mark.gpu
K = 1024


def _rows(L, R, seed, n_random=40):
    C = L // (2 * R)
    edges = [c * C + d for c in range(2 * R) for d in (0, C - 1)]
    rng = np.random.default_rng(seed)
    rows = np.concatenate([np.arange(4), np.arange(L - 4, L), edges, rng.integers(0, L, n_random)])
    return np.unique(rows)


@pytest.mark.parametrize("name,L,hc,kv,U,R,causal", [
    ("bench_c3_1gpu", 128 * K, 32, 8, 1, 1, True),   # the bench line's workload
    ("c3_ring8", 128 * K, 32, 8, 1, 8, True),        # pure ring, zigzag
    ("c4_u4r2", 208 * K, 32, 8, 4, 2, True),         # the paper's headline shape
    ("c5_kv4_u4r2", 128 * K, 32, 4, 4, 2, True),     # GQA kv 4: Ulysses capped at 4
    ("c2_u8_causal", 32 * K, 32, 8, 8, 1, True),     # pure Ulysses
    ("c2_u8_full", 32 * K, 32, 8, 8, 1, False),
])
def test_full_size_sampled_rows(cuda, name, L, hc, kv, U, R, causal):
    hs = 128
    g = torch.Generator(device=cuda).manual_seed(L + 31 * U + R)
    q = (torch.rand(1, L, hc, hs, device=cuda, generator=g) * 2 - 1).to(torch.bfloat16)
    k = (torch.rand(1, L, kv, hs, device=cuda, generator=g) * 2 - 1).to(torch.bfloat16)
    v = (torch.rand(1, L, kv, hs, device=cuda, generator=g) * 2 - 1).to(torch.bfloat16)
    c = UspCase(seq=L, hc=hc, kv_hc=kv, hs=hs, ulysses=U, ring=R, causal=causal)
    out, lses, engines, comm = run_usp_gpu(c, q, k, v, cuda)
    rows = _rows(L, R, seed=L)
    ref_o, ref_l = Oracle.softmax_rows(widen(q[:, rows]), widen(k), widen(v), causal, rows, np.arange(L))
    eo = errors(widen(out[:, rows]), ref_o)
    # LSE: row p lives on ring coordinate r whose ring list holds p, at its
    # index there, heads [u*hc/U, (u+1)*hc/U) on rank r*U + u
    hl = hc // U
    got_l = np.empty_like(ref_l)
    for r in range(R):
        hp = np.asarray(engines[r * U].head_positions())
        where = {int(p): i for i, p in enumerate(hp)}
        for j, p in enumerate(rows):
            if int(p) in where:
                for u in range(U):
                    got_l[0, j, u * hl:(u + 1) * hl] = lses[r * U + u][0, where[int(p)]].double().cpu().numpy()
    el = errors(got_l, ref_l)
    print(f"{name}: rows={len(rows)} O {eo} LSE {el}")
    assert np.isfinite(widen(out[:, rows])).all()
    assert eo["max_abs"] <= O_TOL and el["max_abs"] <= LSE_TOL, (name, eo, el)
    assert all(e.last_launches() >= 1 for e in engines)
    for e in engines:
        e.close()
    if comm is not None:
        comm.close()
