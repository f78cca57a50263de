#!/usr/bin/env python
"""Pipelined Ulysses exchange on one GPU (development aid).

Runs a U x 1 local world (one host thread per rank, the in-process transport:
the all-to-alls are copy-engine transfers on each rank's comm stream) at the
c2 head shape and prints, per chunk count, the per-stage times of rank 0
(usp_engine_stage_times): the exposed waits for the Q/K/V chunks (wait_in.c,
or a2a_in unchunked), the attention launches, and the exposed O exchange
(a2a_out). Every rank shares the one GPU, so absolute times are not a
scaling measurement — the point is which exchanges stay exposed.

    python tools/a2a_overlap.py [L] [U]
    python tools/a2a_overlap.py --host [L] [U]   # usp_attn_fwd_host wall time per call

--host: every rank calls forward_host (pinned host Q/K/V/O/LSE) from its own
thread; the wall time of the whole world per call, chunked exchanges
(fwd_host_a2a: per-chunk upload/pack/exchange and exchange/unpack/download)
against 1 chunk (whole-shard copies around the forward).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_07719_b200 import Comm, ProcessMesh, UspAttention, local_world_forward  # noqa: E402


def run(L, U, chunks, iters=5):
    dev = torch.device("cuda", 0)
    mesh = ProcessMesh(U, 1)
    comm = Comm.local(U)
    engs = [UspAttention(mesh, rank=r, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True, comm=comm)
            for r in range(U)]
    for e in engs:
        e.set_a2a_chunks(chunks)
    qs = [torch.randn(e.q_shape(), device=dev, dtype=torch.bfloat16) for e in engs]
    ks = [torch.randn(e.kv_shape(), device=dev, dtype=torch.bfloat16) for e in engs]
    vs = [torch.randn(e.kv_shape(), device=dev, dtype=torch.bfloat16) for e in engs]
    outs, lses = zip(*[e.alloc_outputs() for e in engs])
    streams = [torch.cuda.Stream(dev) for _ in engs]
    for _ in range(2):
        local_world_forward(engs, qs, ks, vs, outs, lses, streams)
    torch.cuda.synchronize()
    for e in engs:
        e.enable_timing(True)
    for _ in range(iters):
        local_world_forward(engs, qs, ks, vs, outs, lses, streams)
    torch.cuda.synchronize()
    st = {x["stage"]: round(x["ms_total"] / iters, 4) for x in engs[0].stage_times()}
    for e in engs:
        e.close()
    comm.close()
    return st


def run_host(L, U, chunks, iters=5):
    import threading
    import time

    mesh = ProcessMesh(U, 1)
    comm = Comm.local(U)
    engs = [UspAttention(mesh, rank=r, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True, comm=comm)
            for r in range(U)]
    for e in engs:
        e.set_a2a_chunks(chunks)
    pin = lambda s, dt=torch.bfloat16: torch.randn(s, dtype=torch.float32).to(dt).pin_memory()  # noqa: E731
    io = [(pin(e.q_shape()), pin(e.kv_shape()), pin(e.kv_shape()), pin(e.q_shape()),
           pin(tuple(e.alloc_outputs()[1].shape), torch.float32)) for e in engs]

    def world():
        th = [threading.Thread(target=lambda i=i: engs[i].forward_host(*io[i])) for i in range(U)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()

    for _ in range(2):
        world()
    t0 = time.perf_counter()
    for _ in range(iters):
        world()
    ms = (time.perf_counter() - t0) * 1e3 / iters
    h2d = sum(x.numel() * x.element_size() for x in io[0][:3]) * U
    for e in engs:
        e.close()
    comm.close()
    return {"ms_per_call": round(ms, 3), "h2d_bytes_all_ranks": h2d}


if __name__ == "__main__":
    if sys.argv[1:2] == ["--host"]:
        sys.argv.pop(1)
        L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
        U = int(sys.argv[2]) if len(sys.argv) > 2 else 2
        for c in (1, 2, 4):
            print(json.dumps({"L": L, "U": U, "chunks": c, "host": run_host(L, U, c)}), flush=True)
        sys.exit(0)
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    U = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for c in (1, 2, 4):
        print(json.dumps({"L": L, "U": U, "chunks": c, "stages_ms_rank0": run(L, U, c)}), flush=True)
