"""Back-to-back usp_attn_fwd_host calls: per-call GPU time (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True)
pin = lambda shape, dt: torch.randn(shape, dtype=torch.float32).to(dt).pin_memory()  # noqa: E731
q, k, v = pin(eng.q_shape(), torch.bfloat16), pin(eng.kv_shape(), torch.bfloat16), pin(eng.kv_shape(), torch.bfloat16)
o = torch.empty(eng.q_shape(), dtype=torch.bfloat16).pin_memory()
lse = torch.empty(eng.lse_shape(), dtype=torch.float32).pin_memory()
eng.forward_host(q, k, v, o, lse)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
ev[0].record()
t0 = time.perf_counter()
host = []
for i in range(4):
    a = time.perf_counter()
    eng.forward_host(q, k, v, o, lse)
    host.append((time.perf_counter() - a) * 1e3)
    ev[i + 1].record()
torch.cuda.synchronize()
print("per call GPU ms:", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(4)])
print("host enqueue ms:", [round(x, 3) for x in host])
dq, dk, dv = (torch.empty_like(x).cuda() for x in (q, k, v))
do, dl = torch.empty_like(o).cuda(), torch.empty_like(lse).cuda()
dq.copy_(q); dk.copy_(k); dv.copy_(v)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(4):
    eng.forward(dq, dk, dv, do, dl)
e.record(); torch.cuda.synchronize()
print("device forward ms:", round(s.elapsed_time(e) / 4, 3))
