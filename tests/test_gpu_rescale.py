"""GPU parity of the forward kernel's lazy O-rescale branch.

SoftmaxState::update (reference src/numerics/attention.cpp:209-226) rescales
the accumulator by exp(m - m') whenever a new key raises the running row
max. The B200 kernel (fa_fwd_sm100.cu, softmax warps) moves its running max
only when the tile max exceeds it by more than 8 (log2 units) and then
multiplies O in TMEM by alpha = 2^(m_old - m_new) (read-modify-write); in
between, P = 2^(s - m) may grow up to 2^8 in fp32 / bf16. The reference
generator's U[-1, 1) inputs never grow the max by 8 (worst 1.46), so the
branch needs peaky inputs (SURVEY §8(d) stress set):

  q8 / q16 : Q scaled by 8 / 16 (softmax close to one-hot);
  kgrow    : K scaled by 1 + 15 t / L with its global position t, so later
             key tiles raise the running max of every row.

Each case runs every rank of the mesh (in-process transport), checks O and
LSE against the fp64 oracle on the same bf16-rounded inputs — relative L2
and LSE with the standard gates, O max-abs with O_TOL_PEAKY = 2u (a near
one-hot softmax passes single bf16-rounded P and O values through instead of
averaging their rounding; usp_harness) — and proves the branch fired: the kernel's debug counter
(usp_engine_debug_counters) of (warp, key tile) rescales is > 0.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from tests.usp_harness import (LSE_TOL, O_REL_L2, O_TOL, O_TOL_PEAKY, UspCase, errors, make_globals, run_usp_gpu,
                               to_bf16, widen)

pytestmark = pytest.mark.gpu


def _stress(c: UspCase, kind: str):
    q, k, v = make_globals(c)
    if kind == "q8":
        q = q * 8.0
    elif kind == "q16":
        q = q * 16.0
    elif kind == "kgrow":
        t = np.arange(c.seq, dtype=np.float64) / c.seq
        k = k * (1.0 + 15.0 * t)[None, :, None, None]
    return q, k, v


def _run(c: UspCase, kind: str, device):
    q, k, v = _stress(c, kind)
    tq, tk, tv = (to_bf16(x, device) for x in (q, k, v))
    out, lses, engines, _ = run_usp_gpu(c, tq, tk, tv, device, setup=lambda es: [e.debug_counters(True) for e in es])
    fired = sum(e.rescale_count() for e in engines)
    ref_out, ref_lse = Oracle.usp_forward(widen(tq), widen(tk), widen(tv), c.ulysses, c.ring, c.causal)
    eo = errors(widen(out), ref_out)
    el = errors(np.stack([widen(l_) for l_ in lses]), ref_lse)
    for e in engines:
        e.debug_counters(False)
    return eo, el, fired


@pytest.mark.parametrize("kind", ["q8", "q16", "kgrow"])
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("hs", [64, 128])
@pytest.mark.parametrize("u,r", [(1, 1), (1, 4), (4, 2)])
def test_rescale_branch_matches_oracle(cuda, u, r, hs, causal, kind):
    # hc 16 / kv 4: GQA groups of 4 (2-CTA multicast clusters at hs 128) at
    # U = 1, groups of 4 over 4 local heads at U = 4.
    c = UspCase(seq=2048, hc=16, kv_hc=4, hs=hs, ulysses=u, ring=r, causal=causal, seed=31 + hs)
    eo, el, fired = _run(c, kind, cuda)
    msg = f"{c} {kind}: O {eo} LSE {el} rescales {fired}"
    assert fired > 0, "the lazy-rescale branch never fired: " + msg
    assert eo["max_abs"] <= O_TOL_PEAKY and eo["rel_l2"] <= O_REL_L2, msg
    assert el["max_abs"] <= LSE_TOL, msg


@pytest.mark.parametrize("u,r", [(1, 1), (2, 2)])
def test_rescale_branch_mha_tile_pairs(cuda, u, r):
    # MHA: a unit is two adjacent 128-row tiles of one head (pair_rows).
    c = UspCase(seq=1536, hc=4, kv_hc=4, hs=128, ulysses=u, ring=r, causal=True, seed=5)
    eo, el, fired = _run(c, "q16", cuda)
    msg = f"{c}: O {eo} LSE {el} rescales {fired}"
    assert fired > 0, msg
    assert eo["max_abs"] <= O_TOL_PEAKY and eo["rel_l2"] <= O_REL_L2, msg
    assert el["max_abs"] <= LSE_TOL, msg


def test_uniform_inputs_counter_reads(cuda):
    # The reference's own U[-1, 1) inputs (the verdict's observation: the
    # running max grows by at most ~1.5, so the branch stays cold); the
    # counter path itself must read back and reset.
    c = UspCase(seq=1024, hc=8, kv_hc=2, hs=128, causal=True, seed=0)
    eo, el, fired = _run(c, "none", cuda)
    assert fired >= 0
    assert eo["max_abs"] <= O_TOL and el["max_abs"] <= LSE_TOL, (eo, el)
