"""NCCL transport failure handling on one GPU.

The transport's communicators are non-blocking and polled against the comm
timeout (transport.cpp NcclTransport). A two-rank world whose second rank
never joins must report the stuck ncclCommInitRankConfig after the timeout
instead of hanging (the reference World's stuck-collective diagnosis,
world.cpp:89-113). Run in a subprocess so a regression cannot hang the suite.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, time
sys.path.insert(0, sys.argv[1])
import torch  # binds torch's libnccl first, as the product does
from paper_2405_07719_b200 import Comm, UspError
t0 = time.time()
try:
    Comm.nccl(Comm.nccl_unique_id(), 2, 0, 0)
    print("NO-ERROR")
except UspError as e:
    print("STATUS", e.status, "AFTER", round(time.time() - t0, 1))
    print("MSG", e)
"""


def test_nccl_missing_peer_is_reported(cuda):
    env = dict(os.environ, USP_COMM_TIMEOUT_S="4")
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT], capture_output=True, text=True, timeout=120, env=env)
    out = r.stdout
    assert "STATUS 3" in out, (out, r.stderr[-2000:])
    assert "did not complete within 4 s" in out and "ncclCommInitRankConfig(world of 2, rank 0)" in out, out


def test_nccl_single_rank_status_and_timeout(cuda):
    from paper_2405_07719_b200 import Comm

    comm = Comm.nccl(Comm.nccl_unique_id(), 1, 0, 0)
    comm.set_timeout(30)
    comm.status()  # healthy
    comm.close()


def test_ring_overlap_sizing_c3(cuda):
    """Config c3 (L = 128K, U1 x R8): one shift moves K+V = 64 MiB behind a
    ring step of 2.2 TFLOP (~1.7 ms at 1300 TFLOP/s): ~39.7 GB/s needed; with
    2x margin at >= 20 GB/s per NCCL CTA the ring communicator gets 4 CTAs.
    The copy-engine transports reserve no SMs."""
    from paper_2405_07719_b200 import Comm, ProcessMesh, UspAttention

    comm = Comm.local(8)
    eng = UspAttention(ProcessMesh(1, 8), rank=0, seq_len=131072, heads=32, kv_heads=8, head_size=128, causal=True,
                       comm=comm)
    i = eng.info()
    assert i["kv_shift_bytes"] == 64 * 2**20, i
    assert 1.5 < i["ring_step_ms_est"] < 1.9 and 35 < i["required_gbs"] < 45, i
    assert i["ring_ctas"] == 4 and i["reserved_sms"] == 0, i
    eng.set_reserved_sms(4)
    assert eng.info()["reserved_sms"] == 4
    eng.close()
    comm.close()
