"""Minimal backward loop for ncu captures: python tools/profile_bwd.py L [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_07719_b200 import ProcessMesh, UspAttention

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True)
q = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
k = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
v = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
do = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
fwd = eng.forward(q, k, v)
dq, dk, dv = eng.alloc_grads()
for _ in range(iters):
    eng.backward(fwd, do, dq, dk, dv)
torch.cuda.synchronize()
print("done", L, iters)
