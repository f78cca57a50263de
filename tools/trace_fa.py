"""Runs one forward with USP_FA_TRACE=1 and prints the per-tile timeline of CTA 0.
events: 0-4 softmax A (S seen, S loaded, max, exp done, P arrived); 5-9 softmax B;
10/11 MMA (P_A seen, PV_A+QK_A issued); 12/13 (P_B seen, PV_B+QK_B issued)."""
import ctypes, os, sys
os.environ["USP_FA_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2405_07719_b200 import ProcessMesh, UspAttention
from paper_2405_07719_b200._lib import lib
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True)
dev = torch.device("cuda", 0)
q = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
k = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
v = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
o, lse = eng.alloc_outputs()
for _ in range(3): eng.forward(q, k, v, o, lse)
torch.cuda.synchronize()
buf = np.zeros(16 * 256, np.uint64)
assert lib().usp_engine_trace_copy(eng._h, buf.ctypes.data_as(ctypes.c_void_p)) == 1
t = buf.reshape(16, 256).astype(np.int64)
base = t[0, 1]
names = ["A:S", "A:ld", "A:max", "A:exp", "A:P", "B:S", "B:ld", "B:max", "B:exp", "B:P", "M:PA", "M:issA", "M:PB", "M:issB", "S:K", "S:free"]
print("tile " + " ".join(f"{n:>7}" for n in names))
for i in range(2, 40):
    print(f"{i:4d} " + " ".join(f"{(t[e, i] - base) if t[e, i] else -1:7d}" for e in range(16)))
d = lambda a, b: np.median((t[b, 4:200] - t[a, 4:200]))
print("median A: S->ld %.0f ld->max %.0f max->exp %.0f exp->P %.0f | period A %.0f" % (d(0, 1), d(1, 2), d(2, 3), d(3, 4), np.median(np.diff(t[0, 4:200]))))
print("median B: S->ld %.0f ld->max %.0f max->exp %.0f exp->P %.0f" % (d(5, 6), d(6, 7), d(7, 8), d(8, 9)))
print("median P_A arrive->MMA sees %.0f ; MMA sees->issued %.0f ; issued->next S_A seen %.0f" % (
    np.median(t[10, 4:200] - t[4, 4:200]), np.median(t[11, 4:200] - t[10, 4:200]), np.median(t[0, 5:201] - t[11, 4:200])))
print("median S warp: K_j landed -> S_A(j) buffer free %.0f ; S_A(j) seen by softmax - buffer free %.0f ; "
      "A:P(j-1) stored -> K_j landed %.0f" % (np.median(t[15, 4:200] - t[14, 4:200]), np.median(t[0, 4:200] - t[15, 4:200]),
                                            np.median(t[14, 4:200] - t[4, 3:199])))
