"""Minimal forward loop for ncu captures: python tools/profile_target.py L [iters] [causal]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_07719_b200 import ProcessMesh, UspAttention

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
causal = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
dev = torch.device("cuda", 0)
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=causal)
q = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
k = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
v = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
o, lse = eng.alloc_outputs()
for _ in range(iters):
    eng.forward(q, k, v, o, lse)
torch.cuda.synchronize()
print("done", L, iters, causal)
