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


if __name__ == "__main__":
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    U = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for c in (1, 2, 4):
        print(json.dumps({"L": L, "U": U, "chunks": c, "stages_ms_rank0": run(L, U, c)}), flush=True)
