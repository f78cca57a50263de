"""Generates tests/golden/reference_golden.npz from the REFERENCE ITSELF.

Runs the reference's own sources (oracle/_ref/libuspref.so, compiled from
/root/reference/proj/src by oracle/Makefile) on the reference test-suite
cases and stores inputs-by-seed + outputs, so the oracle can be pinned on
hosts where /root/reference does not exist (the GPU box).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference, reference_attention_grad, reference_usp_fwd_bwd  # noqa: E402

# (name, bs, seq, hc, kv, hs, U, R, causal, seed) — the reference test cases
CASES = [
    ("harness_default", 1, 8, 2, 2, 4, 1, 1, False, 1234),      # usp_harness.hpp:16-21
    ("ring_r1_full", 1, 8, 2, 1, 4, 1, 1, False, 501),          # test_usp.cpp:188-236
    ("ring_r1_causal", 1, 8, 2, 1, 4, 1, 1, True, 501),
    ("ring_r2_full", 1, 8, 2, 1, 4, 1, 2, False, 502),
    ("ring_r4_causal", 1, 16, 2, 1, 4, 1, 4, True, 504),
    ("ring_r4_full", 1, 16, 2, 1, 4, 1, 4, False, 504),
    ("fact_1x8_causal", 1, 32, 8, 8, 4, 1, 8, True, 4242),      # test_usp.cpp:315-341
    ("fact_2x4_causal", 1, 32, 8, 8, 4, 2, 4, True, 4242),
    ("fact_4x2_causal", 1, 32, 8, 8, 4, 4, 2, True, 4242),
    ("fact_8x1_causal", 1, 32, 8, 8, 4, 8, 1, True, 4242),
    ("fact_2x4_full", 1, 32, 8, 8, 4, 2, 4, False, 4242),
    ("fact_8x1_full", 1, 32, 8, 8, 4, 8, 1, False, 4242),
    ("gqa_2x2_bs2", 2, 16, 8, 2, 4, 2, 2, True, 999),           # test_usp.cpp:343-362
    ("llama_small_4x2", 1, 64, 32, 8, 8, 4, 2, True, 0),
]


def gen(seed, bs, seq, hc, kv, hs):
    nq, nk = bs * seq * hc * hs, bs * seq * kv * hs
    g = Reference.uniform(seed, nq + 2 * nk)
    return (g[:nq].reshape(bs, seq, hc, hs), g[nq:nq + nk].reshape(bs, seq, kv, hs),
            g[nq + nk:].reshape(bs, seq, kv, hs))


def gen_with_dout(seed, bs, seq, hc, kv, hs):
    """Q, K, V, dO from one stream in that order (commands.cpp:90-102)."""
    nq, nk = bs * seq * hc * hs, bs * seq * kv * hs
    g = Reference.uniform(seed, 2 * nq + 2 * nk)
    return (g[:nq].reshape(bs, seq, hc, hs), g[nq:nq + nk].reshape(bs, seq, kv, hs),
            g[nq + nk:nq + 2 * nk].reshape(bs, seq, kv, hs), g[nq + 2 * nk:].reshape(bs, seq, hc, hs))


def main():
    assert Reference.available(), "reference library not built (needs /root/reference)"
    out = {}
    for name, bs, seq, hc, kv, hs, U, R, causal, seed in CASES:
        q, k, v = gen(seed, bs, seq, hc, kv, hs)
        o, lse, _ = Reference.usp_forward(q, k, v, U, R, causal)
        # the reference World's communication ledger of that forward
        out[f"{name}/ledger"] = np.array(json.dumps(Reference.last_ledger()))
        out[f"{name}/meta"] = np.array([bs, seq, hc, kv, hs, U, R, int(causal), seed], np.int64)
        out[f"{name}/out"] = o
        out[f"{name}/lse"] = lse
        out[f"{name}/ref_attn"] = Reference.reference_attention(q, k, v, causal)
    # backward (usp_attention_backward, usp_attention.cpp:68-89) on the same cases
    for name, bs, seq, hc, kv, hs, U, R, causal, seed in CASES:
        q, k, v, do = gen_with_dout(seed, bs, seq, hc, kv, hs)
        dq, dk, dv = reference_usp_fwd_bwd(q, k, v, do, U, R, causal)
        out[f"{name}/bwd_ledger"] = np.array(json.dumps(Reference.last_ledger()))
        out[f"{name}/bwd_dq"], out[f"{name}/bwd_dk"], out[f"{name}/bwd_dv"] = dq, dk, dv
        g = reference_attention_grad(q, k, v, do, causal)
        out[f"{name}/grad_dq"], out[f"{name}/grad_dk"], out[f"{name}/grad_dv"] = g
    # scrambled positions (test_numerics.cpp:105-117)
    q, k, v = gen(13, 1, 8, 2, 2, 4)
    pos = np.array([3, 0, 7, 4, 1, 6, 2, 5], np.int64)
    out["scrambled/pos"] = pos
    out["scrambled/out"] = Reference.reference_attention(q, k, v, True, pos)
    o, l_ = Reference.softmax_rows(q, k, v, True, pos, pos)
    out["scrambled/sm_out"], out["scrambled/sm_lse"] = o, l_
    out["uniform/seed0"] = Reference.uniform(0, 64)
    out["uniform/seed4242"] = Reference.uniform(4242, 64)
    out["zigzag/16_4"] = Reference.zigzag_partition(16, 4)
    out["zigzag/4096_8"] = Reference.zigzag_partition(4096, 8)
    out["positions/2x2_8"] = np.stack([Reference.positions_for(2, 2, 8, True, r) for r in range(4)])
    out["positions/4x2_64"] = np.stack([Reference.positions_for(4, 2, 64, True, r) for r in range(8)])
    out["positions/2x2_8_even"] = np.stack([Reference.positions_for(2, 2, 8, False, r) for r in range(4)])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
