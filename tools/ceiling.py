#!/usr/bin/env python
"""Practical ceiling for the forward (and, with --bwd, the backward) kernels: library attention kernels on the
same box at the bench shape (verdict r1 item 6).

Causal attention, hc 32 / kv 8 (GQA) / hs 128, bf16, bs 1, at L = 128K (and
32K), TFLOP/s counted like bench.py (4 * hc * hs * L(L+1)/2). Each backend runs
in its own subprocess (a library that JIT-compiles or fails cannot take the
others down); CUDA events over the kernel call, after warm-up, median of 5.

  cudnn     torch SDPA, SDPBackend.CUDNN_ATTENTION (K/V expanded to 32 heads
            if the backend rejects enable_gqa)
  trtllm    flashinfer.prefill.trtllm_batch_context_with_kv_cache (the
            TensorRT-LLM Blackwell FMHA cubins shipped in flashinfer_cubin;
            paged K/V, page 64, HND)
  fa2       flash_attn 2.8 flash_attn_func (sm80 kernels recompiled for sm100)
  ours      this repo's usp_attn_fwd (U = R = 1)
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def flops(L, hc=32, hs=128):
    return 4.0 * hc * hs * L * (L + 1) / 2


def bench(fn, reps=5, warm=2):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def run(backend, L, bwd=False):
    import torch

    dev = torch.device("cuda", 0)
    hc, kv, hs = 32, 8, 128
    g = torch.Generator(device=dev).manual_seed(0)
    u = lambda *s: (torch.rand(s, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, k, v = u(L, hc, hs), u(L, kv, hs), u(L, kv, hs)
    note = ""
    if backend == "cudnn":
        from torch.nn.attention import SDPBackend, sdpa_kernel

        qt, kt, vt = (x.transpose(0, 1).unsqueeze(0) for x in (q, k, v))  # (1, H, L, D)
        try:
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                torch.nn.functional.scaled_dot_product_attention(qt[:, :, :256], kt[:, :, :256], vt[:, :, :256],
                                                                 is_causal=True, enable_gqa=True)
            gqa = True
        except Exception as e:  # noqa: BLE001
            gqa, note = False, f"enable_gqa rejected ({type(e).__name__}); K/V expanded to {hc} heads"
            kt = kt.repeat_interleave(hc // kv, dim=1)
            vt = vt.repeat_interleave(hc // kv, dim=1)

        if bwd:
            qt, kt, vt = (x.contiguous().requires_grad_(True) for x in (qt, kt, vt))
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                out = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=gqa)
            do = torch.rand_like(out) * 2 - 1

            def fn():
                with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                    torch.autograd.grad(out, (qt, kt, vt), do, retain_graph=True)
        else:
            def fn():
                with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                    torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=gqa)
    elif backend == "trtllm":
        if bwd:
            raise SystemExit("trtllm: forward only")
        from flashinfer.prefill import trtllm_batch_context_with_kv_cache

        page = 64
        npages = L // page
        kc = k.view(npages, page, kv, hs).transpose(1, 2).contiguous()  # [pages, kv, page, hs] (HND)
        vc = v.view(npages, page, kv, hs).transpose(1, 2).contiguous()
        ws = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
        bt = torch.arange(npages, dtype=torch.int32, device=dev).view(1, -1)
        seq = torch.tensor([L], dtype=torch.int32, device=dev)
        cq = torch.tensor([0, L], dtype=torch.int32, device=dev)
        out = torch.empty_like(q)

        def fn():
            trtllm_batch_context_with_kv_cache(q, (kc, vc), ws, bt, seq, L, L, 1.0 / hs ** 0.5, 1.0, 1, cq, cq,
                                               out=out, kv_layout="HND", causal=True)
    elif backend == "fa2":
        from flash_attn import flash_attn_func

        qb, kb, vb = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
        if bwd:
            qb, kb, vb = (x.contiguous().requires_grad_(True) for x in (qb, kb, vb))
            out = flash_attn_func(qb, kb, vb, causal=True)
            do = torch.rand_like(out) * 2 - 1

            def fn():
                torch.autograd.grad(out, (qb, kb, vb), do, retain_graph=True)
        else:
            def fn():
                flash_attn_func(qb, kb, vb, causal=True)
    elif backend == "ours":
        from paper_2405_07719_b200 import ProcessMesh, UspAttention

        eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True)
        qo, ko, vo = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
        o, lse = eng.alloc_outputs()
        if bwd:
            fwd = eng.forward(qo, ko, vo)
            do = u(L, hc, hs).unsqueeze(0)
            dq, dk, dv = eng.alloc_grads()

            def fn():
                eng.backward(fwd, do, dq, dk, dv)
        else:
            def fn():
                eng.forward(qo, ko, vo, o, lse)
    else:
        raise SystemExit(f"unknown backend {backend}")
    ms = bench(fn)
    # backward: algorithmic FLOPs = 2.5x the forward's (five GEMMs per visible pair)
    f = flops(L) * (2.5 if bwd else 1.0)
    return {"backend": backend, "pass": "bwd" if bwd else "fwd", "L": L, "ms": ms, "tflops": f / ms / 1e9,
            "note": note}


def main():
    bwd = "--bwd" in sys.argv
    args = [a for a in sys.argv[1:] if a != "--bwd"]
    if len(args) > 1 and args[0] == "--one":
        print("RESULT " + json.dumps(run(args[1], int(args[2]), bwd)), flush=True)
        return
    for L in (131072, 32768):
        for b in ("ours", "cudnn", "fa2") if bwd else ("ours", "cudnn", "trtllm", "fa2"):
            try:
                r = subprocess.run([sys.executable, os.path.abspath(__file__), "--one", b, str(L)] + (["--bwd"] if bwd else []),
                                   capture_output=True, text=True, timeout=600)
                line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
                if line:
                    print(line[0][7:], flush=True)
                else:
                    print(json.dumps({"backend": b, "L": L, "error": (r.stderr or r.stdout)[-600:]}), flush=True)
            except subprocess.TimeoutExpired:
                print(json.dumps({"backend": b, "L": L, "error": "timeout"}), flush=True)


if __name__ == "__main__":
    main()
