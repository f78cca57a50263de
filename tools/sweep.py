"""Every valid ulysses x ring factorisation of the BASELINE configurations at
N = 1, 2, 4, 8 GPUs, one bench.py run each,
collected as JSON lines.

    python tools/sweep.py --gpus 1 2 4 8 --out sweep.jsonl          # a multi-GPU node
    USP_BENCH_SAME_DEVICE=1 python tools/sweep.py --gpus 2 4 --quick  # plumbing check on one GPU

Validity follows the reference's rules (partition.cpp:78-92,
usp_attention.cpp:22-34): U | kv heads, U | q heads, L % 2R == 0 (causal
zigzag), (L / R) % U == 0. Each run is launched like the driver launches
bench.py (torchrun, one process per GPU, 127.0.0.1 rendezvous).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
K = 1024
# (name, L, hc, kv, hs, causal) — BASELINE.json configs[1..4]
CONFIGS = [
    ("c2_llama_32k", 32 * K, 32, 8, 128, True),
    ("c3_llama_128k", 128 * K, 32, 8, 128, True),
    ("c4_llama_208k", 208 * K, 32, 8, 128, True),
    ("c5_kv4_128k", 128 * K, 32, 4, 128, True),
]


def valid(n, u, L, hc, kv, causal):
    r = n // u
    return (n % u == 0 and kv % u == 0 and u <= kv and hc % u == 0 and L % (2 * r if causal else r) == 0
            and (L // r) % u == 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--configs", nargs="+", default=[c[0] for c in CONFIGS])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--transport", default="nccl", choices=["nccl", "p2p"])
    ap.add_argument("--quick", action="store_true", help="L = 32K for every config (plumbing checks)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    port = 29600
    with open(a.out, "a") as out:
        for name, L, hc, kv, hs, causal in CONFIGS:
            if name not in a.configs:
                continue
            if a.quick:
                L = 32 * K
            for n in a.gpus:
                for u in [x for x in (1, 2, 4, 8) if x <= n]:
                    if not valid(n, u, L, hc, kv, causal):
                        continue
                    port += 1
                    args = ["bench.py", "--gpus", str(n), "--ulysses", str(u), "--seq-len", str(L), "--heads", str(hc),
                            "--kv-heads", str(kv), "--head-size", str(hs), "--steps", str(a.steps), "--warmup",
                            str(a.warmup), "--transport", a.transport, "--skip-cpu-baseline"]
                    if not causal:
                        args.append("--non-causal")
                    cmd = ([sys.executable] + args if n == 1 else
                           [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                            "--master-addr", "127.0.0.1", "--master-port", str(port)] + args)
                    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1800)
                    line = next((x for x in res.stdout.splitlines() if x.startswith("{")), None)
                    rec = {"config": name, "n": n, "ulysses": u, "ring": n // u}
                    if line is None:
                        rec["error"] = (res.stderr or res.stdout)[-400:]
                    else:
                        d = json.loads(line)
                        rec.update(value=d["value"], unit=d["unit"], ms_per_step=d["ms_per_step"],
                                   per_gpu=d["value"] / n, e2e=(d.get("e2e") or {}).get("value"),
                                   clocks=d.get("clocks"))
                    print(json.dumps(rec), flush=True)
                    out.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
