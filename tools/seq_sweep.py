#!/usr/bin/env python
"""Forward and backward throughput across sequence lengths at the Llama-3-8B
layer shape (hc 32 / kv 8 / hs 128, causal, U = R = 1; development aid).
Prints one JSON line per length; uniform [-1, 1) inputs as the bench.
    python tools/seq_sweep.py [L ...]        (SWEEP_HS=64: head size 64)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402


def timed(fn, iters):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def run(L):
    dev = torch.device("cuda", 0)
    hs = int(os.environ.get("SWEEP_HS", "128"))
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=hs, causal=True)
    g = torch.Generator(device=dev).manual_seed(L)
    u = lambda s: (torch.rand(s, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v, do = u(eng.q_shape()), u(eng.kv_shape()), u(eng.kv_shape()), u(eng.q_shape())
    o, lse = eng.alloc_outputs()
    dq, dk, dv = eng.alloc_grads()
    iters = max(3, int(2e11 / (L * L)))
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.25)
    fms = timed(lambda: eng.forward(q, k, v, o, lse), iters)
    fwd = eng.forward(q, k, v)
    bms = timed(lambda: eng.backward(fwd, do, dq, dk, dv), max(2, iters // 3))
    c = clk.stop()
    F = eng.flops()
    out = {"L": L, "hs": hs, "fwd_ms": round(fms, 3), "fwd_tflops": round(F / fms / 1e9, 1), "bwd_ms": round(bms, 3),
           "bwd_tflops_algorithmic": round(2.5 * F / bms / 1e9, 1), "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]}
    eng.close()
    return out


if __name__ == "__main__":
    for L in [int(x) for x in (sys.argv[1:] or ["4096", "8192", "16384", "32768", "65536", "131072", "212992"])]:
        print(json.dumps(run(L)), flush=True)
