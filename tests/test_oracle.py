"""Pins the CPU oracle (oracle/usp_oracle.c) before anything is checked with it.

1. bitwise against the committed golden vectors produced by the reference's
   own code (tests/golden/make_golden.py);
2. bitwise against the reference library itself (oracle/_ref) on random
   cases, when it is available (this container);
3. the reference test suite's known answers (test_numerics.cpp,
   test_usp.cpp), restated.
"""
import os

import numpy as np
import pytest

from oracle.oracle import (Oracle, Reference, oracle_reference_attention_grad, oracle_usp_backward,
                           reference_attention_grad, reference_usp_fwd_bwd)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _gen(seed, bs, seq, hc, kv, hs):
    nq, nk = bs * seq * hc * hs, bs * seq * kv * hs
    g = Oracle.uniform(seed, nq + 2 * nk)
    return (g[:nq].reshape(bs, seq, hc, hs), g[nq:nq + nk].reshape(bs, seq, kv, hs),
            g[nq + nk:].reshape(bs, seq, kv, hs))


def test_uniform_source_matches_reference_stream(golden):
    assert np.array_equal(Oracle.uniform(0, 64), golden["uniform/seed0"])
    assert np.array_equal(Oracle.uniform(4242, 64), golden["uniform/seed4242"])


def test_usp_forward_bitwise_vs_golden(golden):
    names = sorted({k.split("/")[0] for k in golden.files if k.endswith("/meta")})
    assert len(names) >= 10
    for name in names:
        bs, seq, hc, kv, hs, U, R, causal, seed = golden[f"{name}/meta"].tolist()
        q, k, v = _gen(seed, bs, seq, hc, kv, hs)
        out, lse = Oracle.usp_forward(q, k, v, U, R, bool(causal))
        assert np.array_equal(out, golden[f"{name}/out"]), name
        assert np.array_equal(lse, golden[f"{name}/lse"]), name
        ref = Oracle.reference_attention(q, k, v, bool(causal))
        assert np.array_equal(ref, golden[f"{name}/ref_attn"]), name


def test_scrambled_positions_bitwise_vs_golden(golden):
    q, k, v = _gen(13, 1, 8, 2, 2, 4)
    pos = golden["scrambled/pos"]
    assert np.array_equal(Oracle.reference_attention(q, k, v, True, pos), golden["scrambled/out"])
    o, l_ = Oracle.softmax_rows(q, k, v, True, pos, pos)
    assert np.array_equal(o, golden["scrambled/sm_out"])
    assert np.array_equal(l_, golden["scrambled/sm_lse"])


def test_layout_vs_golden(golden):
    assert np.array_equal(Oracle.zigzag_partition(16, 4), golden["zigzag/16_4"])
    assert np.array_equal(Oracle.zigzag_partition(4096, 8), golden["zigzag/4096_8"])
    for key, (U, R, L, zz) in {"positions/2x2_8": (2, 2, 8, True), "positions/4x2_64": (4, 2, 64, True),
                               "positions/2x2_8_even": (2, 2, 8, False)}.items():
        got = np.stack([Oracle.positions_for(U, R, L, zz, r) for r in range(U * R)])
        assert np.array_equal(got, golden[key]), key


@pytest.mark.skipif(not Reference.available(), reason="reference sources not present on this host")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bitwise_vs_reference_library_random(seed):
    rng = np.random.default_rng(seed)
    for _ in range(4):
        U = int(rng.choice([1, 2, 4]))
        R = int(rng.choice([1, 2, 3]))
        kv = U * int(rng.choice([1, 2]))
        hc = kv * int(rng.choice([1, 2, 4]))
        hs = int(rng.choice([3, 4, 8]))
        seq = 2 * R * U * int(rng.integers(1, 5))
        bs = int(rng.choice([1, 2]))
        causal = bool(rng.integers(0, 2))
        q, k, v = _gen(int(rng.integers(0, 1 << 30)), bs, seq, hc, kv, hs)
        o1, l1 = Oracle.usp_forward(q, k, v, U, R, causal)
        o2, l2, _ = Reference.usp_forward(q, k, v, U, R, causal)
        assert np.array_equal(o1, o2) and np.array_equal(l1, l2), (U, R, kv, hc, hs, seq, bs, causal)
        pos = rng.permutation(seq)
        assert np.array_equal(Oracle.reference_attention(q, k, v, causal, pos),
                              Reference.reference_attention(q, k, v, causal, pos))


def _gen_do(seed, bs, seq, hc, kv, hs):
    nq, nk = bs * seq * hc * hs, bs * seq * kv * hs
    g = Oracle.uniform(seed, 2 * nq + 2 * nk)
    return (g[:nq].reshape(bs, seq, hc, hs), g[nq:nq + nk].reshape(bs, seq, kv, hs),
            g[nq + nk:nq + 2 * nk].reshape(bs, seq, kv, hs), g[nq + 2 * nk:].reshape(bs, seq, hc, hs))


def test_backward_bitwise_vs_golden(golden):
    """usp_attention_backward and reference_attention_grad restated
    (oracle/usp_oracle.c) == the reference's own outputs, bit for bit."""
    names = sorted({k.split("/")[0] for k in golden.files if k.endswith("/bwd_dq")})
    assert len(names) >= 10
    for name in names:
        bs, seq, hc, kv, hs, U, R, causal, seed = golden[f"{name}/meta"].tolist()
        q, k, v, do = _gen_do(seed, bs, seq, hc, kv, hs)
        got = oracle_usp_backward(q, k, v, do, U, R, bool(causal))
        for g_, key in zip(got, ("dq", "dk", "dv")):
            assert np.array_equal(g_, golden[f"{name}/bwd_{key}"]), (name, key)
        got = oracle_reference_attention_grad(q, k, v, do, bool(causal))
        for g_, key in zip(got, ("dq", "dk", "dv")):
            assert np.array_equal(g_, golden[f"{name}/grad_{key}"]), (name, key)


@pytest.mark.skipif(not Reference.available(), reason="reference sources not present on this host")
@pytest.mark.parametrize("seed", [5, 6])
def test_backward_bitwise_vs_reference_library_random(seed):
    rng = np.random.default_rng(seed)
    for _ in range(3):
        U = int(rng.choice([1, 2, 4]))
        R = int(rng.choice([1, 2, 3]))
        kv = U * int(rng.choice([1, 2]))
        hc = kv * int(rng.choice([1, 2, 4]))
        hs = int(rng.choice([3, 4, 8]))
        seq = 2 * R * U * int(rng.integers(1, 4))
        bs = int(rng.choice([1, 2]))
        causal = bool(rng.integers(0, 2))
        q, k, v, do = _gen_do(int(rng.integers(0, 1 << 30)), bs, seq, hc, kv, hs)
        a = oracle_usp_backward(q, k, v, do, U, R, causal)
        b = reference_usp_fwd_bwd(q, k, v, do, U, R, causal)
        assert all(np.array_equal(x, y) for x, y in zip(a, b)), (U, R, kv, hc, hs, seq, bs, causal)
        pos = rng.permutation(seq)
        a = oracle_reference_attention_grad(q, k, v, do, causal, pos)
        b = reference_attention_grad(q, k, v, do, causal, pos)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_backward_matches_finite_differences():
    """Known answer independent of the reference: d<dO, O>/dQ by central
    differences on a tiny case."""
    q, k, v, do = _gen_do(77, 1, 6, 2, 1, 3)
    dq, dk, dv = oracle_reference_attention_grad(q, k, v, do, True)
    eps = 1e-6
    for arr, grad in ((q, dq), (k, dk), (v, dv)):
        for idx in [(0, 0, 0, 0), (0, 3, 0, 1), (0, 5, 0, 2)]:
            a0 = arr[idx]
            arr[idx] = a0 + eps
            fp = float((Oracle.reference_attention(q, k, v, True) * do).sum())
            arr[idx] = a0 - eps
            fm = float((Oracle.reference_attention(q, k, v, True) * do).sum())
            arr[idx] = a0
            assert abs((fp - fm) / (2 * eps) - grad[idx]) < 1e-6, idx


# ---- known answers from the reference test suite -------------------------

def test_pinned_two_token_identity():
    # test_numerics.cpp:73-90
    x = np.zeros((1, 2, 1, 2))
    x[0, 0, 0, 0] = 1.0
    x[0, 1, 0, 1] = 1.0
    out = Oracle.reference_attention(x, x, x, False)
    p_match, p_other = 0.6697615493266569, 0.33023845067334307
    np.testing.assert_allclose(out[0, :, 0, :], [[p_match, p_other], [p_other, p_match]], rtol=1e-14)


def test_single_key_output_is_v_exactly():
    # test_numerics.cpp:61-71
    g = Oracle.uniform(7, 3 * 2 * 3 * 4)
    q, k, v = (g[i * 24:(i + 1) * 24].reshape(2, 1, 3, 4) for i in range(3))
    for causal in (False, True):
        assert np.array_equal(Oracle.reference_attention(q, k, v, causal), v)


def test_rows_sum_to_one_with_unit_v():
    # test_numerics.cpp:119-130
    g = Oracle.uniform(17, 2 * 2 * 9 * 3 * 5, -3.0, 3.0)
    q, k = g[:270].reshape(2, 9, 3, 5), g[270:].reshape(2, 9, 3, 5)
    v = np.ones_like(q)
    for causal in (False, True):
        assert np.abs(Oracle.reference_attention(q, k, v, causal) - 1.0).max() < 1e-12


def test_gqa_equals_explicit_replication_bitwise():
    # test_numerics.cpp:132-157
    hc = 4
    for kv in (1, 2):
        q, k, v = _gen(19, 1, 5, hc, kv, 3)
        rep = [h * kv // hc for h in range(hc)]
        for causal in (False, True):
            a = Oracle.reference_attention(q, k, v, causal)
            b = Oracle.reference_attention(q, k[:, :, rep], v[:, :, rep], causal)
            assert np.array_equal(a, b)


def test_zigzag_and_balance():
    # test_usp.cpp:20-61
    assert Oracle.zigzag_partition(16, 4).tolist() == [[0, 1, 14, 15], [2, 3, 12, 13], [4, 5, 10, 11],
                                                       [6, 7, 8, 9]]
    with pytest.raises(ValueError):
        Oracle.zigzag_partition(10, 4)
    assert Oracle.causal_pair_counts(Oracle.even_partition(16, 4), 16).tolist() == [10, 26, 42, 58]
    assert Oracle.causal_pair_counts(Oracle.zigzag_partition(16, 4), 16).tolist() == [34] * 4
    for ring in (1, 2, 3, 4, 8):
        for seq in (2 * ring, 6 * ring, 16 * ring):
            counts = Oracle.causal_pair_counts(Oracle.zigzag_partition(seq, ring), seq)
            assert (counts == seq * (seq + 1) // 2 // ring).all()


def test_shard_spec_positions():
    # test_usp.cpp:68-91
    got = [Oracle.positions_for(2, 2, 8, True, r).tolist() for r in range(4)]
    assert got == [[0, 1], [6, 7], [2, 3], [4, 5]]


def test_usp_equals_reference_attention_across_factorizations():
    # test_usp.cpp:315-341 (O within 1e-12 of the single-device reference)
    q, k, v = _gen(4242, 1, 32, 8, 8, 4)
    for causal in (True, False):
        ref = Oracle.reference_attention(q, k, v, causal)
        for U, R in ((1, 8), (2, 4), (4, 2), (8, 1)):
            out, _ = Oracle.usp_forward(q, k, v, U, R, causal)
            assert np.abs(out - ref).max() < 1e-12


def test_head_limit_rejected():
    # test_usp.cpp:435-454: U=16 > kv=8
    q, k, v = _gen(1, 1, 32, 16, 8, 4)
    with pytest.raises(ValueError):
        Oracle.usp_forward(q, k, v, 16, 1, False)
