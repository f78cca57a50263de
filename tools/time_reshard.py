#!/usr/bin/env python
"""Ulysses pack / unpack throughput: the bulk-copy (TMA
cp.async.bulk) reshard kernel vs the vector-load fallback (USPB_NO_BULK=1).

Runs the whole forward of a U x R mesh on one GPU (in-process transport, one
engine per rank) with stage timing on, and reports rank 0's `pack` (Q, K, V
-> [peer][T][H/U][hs] staging, one launch) and `unpack` (O [peer][T][H/U][hs]
-> (T, H, hs)) stages: ms and GB/s of algorithmic bytes (read + write).

  python tools/time_reshard.py
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [  # name, L, U, R
    ("c2 L32K U8R1", 32768, 8, 1),
    ("c4 L208K U4R2", 212992, 4, 2),
    ("c5 L128K U4R1 kv4", 131072, 4, 1),
]


def one(name, L, U, R):
    import torch

    from paper_2405_07719_b200 import Comm, ProcessMesh, UspAttention, local_world_forward

    dev = torch.device("cuda", 0)
    hc, kv, hs = 32, (4 if "kv4" in name else 8), 128
    mesh = ProcessMesh(U, R)
    n = U * R
    comm = Comm.local(n)
    engs = [UspAttention(mesh, rank=r, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True, comm=comm)
            for r in range(n)]
    T = L // n
    u = lambda s: (torch.rand(s, device=dev) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    qs = [u((1, T, hc, hs)) for _ in engs]
    ks = [u((1, T, kv, hs)) for _ in engs]
    vs = [u((1, T, kv, hs)) for _ in engs]
    outs, lses = zip(*[e.alloc_outputs() for e in engs])
    streams = [torch.cuda.Stream(dev) for _ in engs]
    local_world_forward(engs, qs, ks, vs, outs, lses, streams)
    torch.cuda.synchronize()
    for e in engs:
        e.enable_timing(True)
    reps = 5
    for _ in range(reps):
        local_world_forward(engs, qs, ks, vs, outs, lses, streams)
    torch.cuda.synchronize()
    st = {x["stage"]: x["ms_total"] / x["count"] for x in engs[0].stage_times()}
    qb = T * hc * hs * 2
    kvb = T * kv * hs * 2
    res = {"case": name, "bulk": os.environ.get("USPB_NO_BULK") is None, "stages_ms": st}
    if "pack" in st:
        b = 2 * (qb + 2 * kvb)
        res["pack_gbs"] = b / (st["pack"] * 1e-3) / 1e9
        res["pack_bytes"] = b
    if "unpack" in st:
        b = 2 * qb
        res["unpack_gbs"] = b / (st["unpack"] * 1e-3) / 1e9
    print("RESULT " + json.dumps(res), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        c = CASES[int(sys.argv[2])]
        one(*c)
        return
    for i in range(len(CASES)):
        for bulk in (True, False):
            env = dict(os.environ)
            if not bulk:
                env["USPB_NO_BULK"] = "1"
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--one", str(i)], capture_output=True,
                               text=True, env=env, timeout=600)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
            print(line[0][7:] if line else json.dumps({"case": CASES[i][0], "error": r.stderr[-800:]}), flush=True)


if __name__ == "__main__":
    main()
