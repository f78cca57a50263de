#!/usr/bin/env python
"""Ring-overlap evidence on ONE GPU (verdict r1 item 3).

A c3 ring step (rank tokens 16K, hc 32 / kv 8 / hs 128, 2.2 TFLOP — the
zigzag off-diagonal step of L = 128K on 8 GPUs) is run by the product
attention kernel while a 1-rank NCCL communicator moves the step's K+V
block (64 MiB: self send/recv, NCCL's copy kernel) on a side stream — the
B200 stand-in for the next block's ring shift. For each NCCL CTA cap k the
attention grid leaves k SMs free (usp_engine_set_reserved_sms, as the engine
does for its ring communicator) and NCCL_MAX_CTAS = k. Reported per k:
attention alone / concurrent (CUDA events on its stream), the transfer alone
/ concurrent and its GB/s, and the attention slowdown.

  python tools/overlap_nccl.py            # sweeps k in 1 2 4 8 (one process each)
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(k: int, reps: int = 20):
    import torch
    import torch.distributed as dist

    from paper_2405_07719_b200 import ProcessMesh, UspAttention

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ.get("PORT", "29611"))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    L, hc, kv, hs = 16384, 32, 8, 128
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True)
    eng.set_reserved_sms(k)
    u = lambda shape: (torch.rand(shape, device=dev) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, kk, v = u(eng.q_shape()), u(eng.kv_shape()), u(eng.kv_shape())
    o, lse = eng.alloc_outputs()
    nbytes = 2 * L * kv * hs * 2  # K + V of one ring block (c3: 64 MiB)
    x = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def shift():
        for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, x, 0), dist.P2POp(dist.irecv, y, 0)]):
            r.wait()

    def timed(fn, stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
            fn()
            e1.record()
        return e0, e1

    for _ in range(5):
        eng.forward(q, kk, v, o, lse, sa)
        with torch.cuda.stream(sb):
            shift()
    torch.cuda.synchronize()
    attn_alone, comm_alone, attn_conc, comm_conc = [], [], [], []
    for _ in range(reps):
        a = timed(lambda: eng.forward(q, kk, v, o, lse, sa), sa)
        torch.cuda.synchronize()
        attn_alone.append(a[0].elapsed_time(a[1]))
        c = timed(shift, sb)
        torch.cuda.synchronize()
        comm_alone.append(c[0].elapsed_time(c[1]))
    for _ in range(reps):
        # the transfer starts with the kernel (both streams released together)
        gate = torch.cuda.Event()
        torch.cuda.current_stream().record_event(gate)
        sa.wait_event(gate)
        sb.wait_event(gate)
        a = timed(lambda: eng.forward(q, kk, v, o, lse, sa), sa)
        c = timed(shift, sb)
        torch.cuda.synchronize()
        attn_conc.append(a[0].elapsed_time(a[1]))
        comm_conc.append(c[0].elapsed_time(c[1]))
    med = lambda xs: sorted(xs)[len(xs) // 2]  # noqa: E731
    res = {"nccl_max_ctas": k, "reserved_sms": k, "kv_bytes": nbytes,
           "attn_alone_ms": med(attn_alone), "attn_concurrent_ms": med(attn_conc),
           "attn_slowdown": med(attn_conc) / med(attn_alone) - 1.0,
           "shift_alone_ms": med(comm_alone), "shift_concurrent_ms": med(comm_conc),
           "shift_alone_gbs": nbytes / med(comm_alone) / 1e6, "shift_concurrent_gbs": nbytes / med(comm_conc) / 1e6,
           "step_tflops_alone": eng.flops() / med(attn_alone) / 1e9,
           "hidden": med(comm_conc) < med(attn_conc)}
    print("RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(int(sys.argv[2]))
        return
    rows = []
    for i, k in enumerate((0, 1, 2, 4, 8)):
        # k = 0: no SM left free, the NCCL kernel (1 CTA) queues behind the
        # persistent attention grid
        env = dict(os.environ, NCCL_MAX_CTAS=str(max(k, 1)), NCCL_MIN_CTAS="1", PORT=str(29611 + i))
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--one", str(k)], capture_output=True,
                           text=True, env=env, timeout=600)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        if not line:
            print(r.stdout[-2000:], r.stderr[-3000:], file=sys.stderr)
            continue
        rows.append(json.loads(line[0][7:]))
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"summary": [(r["nccl_max_ctas"], round(r["attn_slowdown"] * 100, 2),
                                   round(r["shift_concurrent_gbs"], 1)) for r in rows],
                      "columns": "nccl_max_ctas, attention slowdown %, concurrent shift GB/s"}))


if __name__ == "__main__":
    main()
