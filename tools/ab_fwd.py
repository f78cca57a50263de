#!/usr/bin/env python
"""A/B device timing of forward- (or, with AB_BWD=1, backward-) kernel builds (development aid).

  python tools/ab_fwd.py [variant ...]      # "" = the product build

Each variant is paper_2405_07719_b200/libusp_b200_<variant>.so (build.py with
USPB_VARIANT), loaded through USPB_LIB_PATH in its own subprocess; rounds
alternate A B A B ... so drift of the power-capped clock hits both alike.
Prints TFLOP/s and the median SM clock of every run at each length.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(L, hs, hc, kv, causal):
    import time

    import torch

    from bench import ClockSampler
    from paper_2405_07719_b200 import ProcessMesh, UspAttention

    dev = torch.device("cuda", 0)
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=causal)
    u = lambda s: (torch.rand(s, device=dev) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v = u(eng.q_shape()), u(eng.kv_shape()), u(eng.kv_shape())
    o, lse = eng.alloc_outputs()
    iters = max(5, int(6e11 / (L * L)))
    bwd = os.environ.get("AB_BWD") == "1"
    if bwd:
        eng.set_deterministic(os.environ.get("AB_DET") == "1")
        fwd = eng.forward(q, k, v, o, lse)
        do = u(eng.q_shape())
        dq, dk, dv = eng.alloc_grads()
        iters = max(3, iters // 3)

    def step():
        if bwd:
            eng.backward(fwd, do, dq, dk, dv)
        else:
            eng.forward(q, k, v, o, lse)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.25)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        step()
    e.record()
    torch.cuda.synchronize()
    c = clk.stop()
    ms = s.elapsed_time(e) / iters
    print("RESULT " + json.dumps({"L": L, "hs": hs, "ms": ms, "tflops": eng.flops() * (2.5 if bwd else 1.0) / ms / 1e9, "pass": "bwd" if bwd else "fwd",
                                  "sm_mhz": c["sm_mhz"], "w": c["power_w_max"]}), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        L, hs, hc, kv, causal = (int(x) for x in sys.argv[2:7])
        child(L, hs, hc, kv, bool(causal))
        return
    variants = sys.argv[1:] or ["", "r01"]
    shapes = [(131072, 128, 32, 8, 1), (32768, 128, 32, 8, 1), (32768, 64, 8, 8, 1), (32768, 128, 32, 8, 0)]
    if os.environ.get("AB_SHAPES") == "long":
        shapes = shapes[:1]
    elif os.environ.get("AB_SHAPES") == "bwd":
        shapes = shapes[:2]
    elif os.environ.get("AB_SHAPES") == "hs64":
        shapes = [(32768, 64, 8, 8, 1), (32768, 64, 32, 8, 1), (131072, 64, 32, 8, 1), (32768, 64, 8, 8, 0)]
    for rnd in range(int(os.environ.get("AB_ROUNDS", "2"))):
        for sh in shapes:
            for var in variants:
                lib = os.path.join(ROOT, "paper_2405_07719_b200", f"libusp_b200_{var}.so" if var else "libusp_b200.so")
                env = dict(os.environ, USPB_LIB_PATH=lib)
                r = subprocess.run([sys.executable, os.path.abspath(__file__), "--child"] + [str(x) for x in sh],
                                   capture_output=True, text=True, env=env, timeout=900)
                line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
                res = json.loads(line[0][7:]) if line else {"error": r.stderr[-500:]}
                res.update(variant=var or "product", round=rnd, shape=sh)
                print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
