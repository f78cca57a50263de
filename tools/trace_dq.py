"""Per-key-tile timeline of the dQ kernel's CTA 0 (development aid; see trace_bwd.py).

events: 0-2 warp half 0 (S seen, dP seen, dS done); 4-6 half 1; 8 S(j+1)
issued, 9 dp_free seen, 10 dP(j+1) issued, 11/12 dS pair 0/1 seen (MMA
warp); 14/15 producer issued K / V of tile j.

    USPB_TRACE_BUILD=1 python -c "import __graft_entry__ as g; g.build()"
    python tools/trace_dq.py [L]
"""
import ctypes
import os
import sys

os.environ["USP_BWD_TRACE"] = "dq"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402
from paper_2405_07719_b200._lib import lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True)
dev = torch.device("cuda", 0)
q = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
k = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
v = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
do = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
fwd = eng.forward(q, k, v)
dq, dk, dv = eng.alloc_grads()
for _ in range(2):
    eng.backward(fwd, do, dq, dk, dv)
torch.cuda.synchronize()
buf = np.zeros(16 * 256, np.uint64)
assert lib().usp_engine_trace_copy(eng._h, buf.ctypes.data_as(ctypes.c_void_p)) == 1
t = buf.reshape(16, 256).astype(np.int64)
names = ["0S", "0dP", "0dS", "-", "1S", "1dP", "1dS", "-", "MSj", "Mfree", "MdPj", "M0", "M1", "-", "TK", "TV"]
base = t[0, 1]
print("tile " + " ".join(f"{n:>7}" for n in names))
for i in range(1, 30):
    print(f"{i:4d} " + " ".join(f"{(t[e, i] - base) if t[e, i] else -1:7d}" for e in range(16)))
ok = [i for i in range(4, 200) if all(t[e, i] for e in (0, 1, 2, 8, 9, 10, 11, 12)) and t[0, i + 1]]


def med(a, b, shift=0):
    return float(np.median([t[b, i + shift] - t[a, i] for i in ok]))


print("period (S seen -> next S seen, half 0): %.0f" % med(0, 0, 1))
print("half 0: S seen->dP seen %.0f | dP seen->dS done %.0f | dS done->next S seen %.0f" % (med(0, 1), med(1, 2), med(2, 0, 1)))
print("MMA: S(j+1) issued->dp_free seen %.0f | ->dP(j+1) issued %.0f | ->pair0 seen %.0f | ->pair1 seen %.0f | pair1->next S issued %.0f"
      % (med(8, 9), med(9, 10), med(10, 11), med(11, 12), med(12, 8, 1)))
print("MMA: dS done(h0) -> pair1 seen %.0f ; S(j+1) issued -> S seen by compute (next tile) %.0f ; dP(j+1) issued -> dP seen %.0f"
      % (med(2, 12), med(8, 0, 1), med(10, 1, 1)))
