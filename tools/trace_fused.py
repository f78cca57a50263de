"""Per-tile timeline of the fused backward kernel's CTA 0 (development aid).

Needs a library built with USPB_TRACE_BUILD=1 (clock64 stamps compiled in);
runs one backward with USP_BWD_TRACE=dkdv and prints, per q tile g, the
stamps relative to the first one and the median intervals.

events: 0-3 warp half 0 (S seen, P done, dP seen, dS stored); 4 half 0 saw
dv_done; 5-7 half 1 (P done, dP seen, dS stored); 8 MMA warp saw P pair 1;
9 S(i+1) issued; 10 saw dS tile; 11 dQ^T + dK issued; 12 half 0 dS computed
(before the dv_done wait); 13 dP(i+1) issued; 14 drain saw dQ^T; 15 drain
handed the last chunk to TMA.

    USPB_TRACE_BUILD=1 python -c "import __graft_entry__ as g; g.build()"
    python tools/trace_fused.py [L]
"""
import ctypes
import os
import sys

os.environ["USP_BWD_TRACE"] = "fused"
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
names = ["0S", "0P", "0dP", "0dS", "0dvd", "1P", "1dP", "1dS", "Mp1", "MSi", "MdS", "MdQK", "0dSc", "MdPi", "Dfull", "Ddone"]
base = t[0, 1]
print("tile " + " ".join(f"{n:>7}" for n in names))
for i in range(1, 30):
    print(f"{i:4d} " + " ".join(f"{(t[e, i] - base) if t[e, i] else -1:7d}" for e in range(16)))
lo, hi = 4, 200
ok = [i for i in range(lo, hi) if all(t[e, i] for e in range(16)) and t[0, i + 1]]


def med(a, b, shift=0):
    return float(np.median([t[b, i + shift] - t[a, i] for i in ok]))


print("period (S seen -> next S seen, half 0): %.0f" % med(0, 0, 1))
print("half 0: S->P done %.0f | P done->dP seen %.0f | dP seen->dS computed %.0f | ->dv_done seen %.0f | ->dS stored %.0f | ->next S %.0f"
      % (med(0, 1), med(1, 2), med(2, 12), med(12, 4), med(4, 3), med(3, 0, 1)))
print("half 1: P done - half 0 P done %.0f | dS stored - half 0 dS stored %.0f" % (med(1, 5), med(3, 7)))
print("MMA: P done(h0)->pair1 seen %.0f | ->S(i+1) issued %.0f | dS stored(h0)->dS seen %.0f | ->dQ,dK issued %.0f"
      % (med(1, 8), med(8, 9), med(3, 10), med(10, 11)))
print("     dQ,dK issued->dP(i+1) issued %.0f | dP(i+1) issued->dP seen by compute %.0f"
      % (med(11, 13), med(13, 2, 1)))
print("drain: dS seen(MMA)->dQ^T seen %.0f | dQ^T seen->all chunks to TMA %.0f"
      % (med(10, 14), med(14, 15)))
