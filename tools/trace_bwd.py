"""Per-q-tile timeline of the dK/dV kernel's CTA 0 (development aid).

Needs a library built with USPB_TRACE_BUILD=1 (clock64 stamps compiled in);
runs one backward with USP_BWD_TRACE=dkdv and prints, per q tile g, the
stamps relative to the first one and the median intervals.

events: 0-3 warp half 0 (S seen, P done, dP seen, dS done); 4-7 half 1;
8/9 MMA warp saw P pair 0/1; 10 S(i+1) issued; 11/12 saw dS pair 0/1;
13 dP(i+1) issued; 14/15 producer issued Q / dO of tile g.

    USPB_TRACE_BUILD=1 python -c "import __graft_entry__ as g; g.build()"
    python tools/trace_bwd.py [L]
"""
import ctypes
import os
import sys

os.environ["USP_BWD_TRACE"] = "dkdv"
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
names = ["0S", "0P", "0dP", "0dS", "1S", "1P", "1dP", "1dS", "Mp0", "Mp1", "MSi", "Md0", "Md1", "MdPi", "TQ", "TdO"]
base = t[0, 1]
print("tile " + " ".join(f"{n:>7}" for n in names))
for i in range(1, 30):
    print(f"{i:4d} " + " ".join(f"{(t[e, i] - base) if t[e, i] else -1:7d}" for e in range(16)))
lo, hi = 4, 200
ok = [i for i in range(lo, hi) if all(t[e, i] for e in range(14)) and all(t[e, i + 1] for e in (0, 4))]


def med(a, b, shift=0):
    return float(np.median([t[b, i + shift] - t[a, i] for i in ok]))


print("period (S seen -> next S seen, half 0): %.0f" % med(0, 0, 1))
print("half 0: S->P done %.0f | P done->dP seen %.0f | dP seen->dS done %.0f | dS done->next S seen %.0f"
      % (med(0, 1), med(1, 2), med(2, 3), med(3, 0, 1)))
print("half 1: S->P done %.0f | P done->dP seen %.0f | dP seen->dS done %.0f | dS done->next S seen %.0f"
      % (med(4, 5), med(5, 6), med(6, 7), med(7, 4, 1)))
print("MMA: P done(h0)->pair1 seen %.0f | pair1 seen->S(i+1) issued %.0f | S(i+1) issued->S seen by compute %.0f"
      % (med(1, 9), med(9, 10), med(10, 0, 1)))
print("MMA: dS done(h0)->dS pair1 seen %.0f | pair1 seen->dP(i+1) issued %.0f | dP(i+1) issued->dP seen %.0f"
      % (med(3, 12), med(12, 13), med(13, 2, 1)))
print("producer: Q(g+2) issued relative to S(g+2) seen: %.0f" % float(np.median([t[0, i + 2] - t[14, i + 2] for i in ok])))
