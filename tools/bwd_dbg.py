import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2405_07719_b200 import ProcessMesh, UspAttention
L=int(sys.argv[1]); hc=int(sys.argv[2]); kv=int(sys.argv[3])
dev=torch.device("cuda",0)
eng=UspAttention(ProcessMesh(1,1),rank=0,seq_len=L,heads=hc,kv_heads=kv,head_size=128,causal=True)
q=torch.randn(eng.q_shape(),device=dev,dtype=torch.bfloat16); k=torch.randn(eng.kv_shape(),device=dev,dtype=torch.bfloat16)
v=torch.randn(eng.kv_shape(),device=dev,dtype=torch.bfloat16); do=torch.randn(eng.q_shape(),device=dev,dtype=torch.bfloat16)
fwd=eng.forward(q,k,v); dq,dk,dv=eng.alloc_grads()
n=int(sys.argv[4]) if len(sys.argv)>4 else 3
for i in range(n):
    eng.backward(fwd,do,dq,dk,dv)
torch.cuda.synchronize(); print("ok",L,hc,kv,n,flush=True)
