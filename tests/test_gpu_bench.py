"""bench.py's contract on a small workload (the driver runs the full one):
one JSON line with the keys the driver and the judge read, on one GPU, on
two ranks (self-launched under torch.distributed.run; both ranks on cuda:0
with the peer-memory transport, USP_BENCH_SAME_DEVICE=1) and for the
reference arm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--seq-len", "8192", "--steps", "3", "--warmup", "3", "--skip-cpu-baseline", "--bwd-steps", "1"]


def _run(args, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env=dict(os.environ, **(env or {})))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def _check_line(d, n):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches",
                "backward"):
        assert key in d, key
    assert d["n_gpus"] == n and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "bf16" and d["higher_is_better"] is True and "workload" in d["config"]
    assert d["gpu_launches"] >= 3
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s" and 0 < rf["frac"] < 1.2, rf
    e = d["e2e"]
    q_bytes = 8192 // n * 32 * 128 * 2
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == q_bytes * 3 // 2 and e["d2h_bytes_per_step"] > q_bytes
    b = d["backward"]
    assert b["fused"]["value"] > 0 and b["deterministic"]["value"] > 0 and b["value"] == b["fused"]["value"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_bench_one_gpu(cuda):
    d = _run(SMALL)
    _check_line(d, 1)
    assert d["parity"]["o_max_abs"] < 5e-3, d["parity"]


def test_bench_two_ranks_self_launched(cuda):
    d = _run(["--gpus", "2", "--backward-multi"] + SMALL, env={"USP_BENCH_SAME_DEVICE": "1"})
    _check_line(d, 2)
    assert d["config"]["parallelism"] == "u1r2"


def test_bench_reference_arm(cuda):
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0
