import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle.oracle import Oracle
from paper_2405_07719_b200 import ProcessMesh, UspAttention
for (L, hc, kv) in ((512, 8, 2), (2048, 32, 8), (1000, 8, 2)):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(L)
    q = (torch.rand(1, L, hc, 128, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    k = (torch.rand(1, L, kv, 128, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    v = (torch.rand(1, L, kv, 128, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=128, causal=True)
    res = eng.forward(q, k, v)
    torch.cuda.synchronize()
    ref = Oracle.reference_attention(q.double().cpu().numpy(), k.double().cpu().numpy(), v.double().cpu().numpy(), True)
    err = np.abs(res.out.double().cpu().numpy() - ref).max()
    print(L, hc, kv, "max|dO|", err, flush=True)
