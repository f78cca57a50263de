import torch, sys
sys.path.insert(0, '.')
from paper_2405_07719_b200 import ProcessMesh, UspAttention
L, hc, kv = 512, 8, 2
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=128, causal=True)
dev = torch.device('cuda', 0)
q = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
k = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
v = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
do = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
f = eng.forward(q, k, v)
g = eng.backward(f, do)
torch.cuda.synchronize()
print("ok", float(g.dq.float().abs().max()))
