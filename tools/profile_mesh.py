"""One hybrid-mesh forward on the in-process transport (ncu target for the
pack/unpack kernels): python tools/profile_mesh.py L U R"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from tests.usp_harness import UspCase, run_usp_gpu  # noqa: E402

L, U, R = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else ("212992", "4", "2")))
dev = torch.device("cuda", 0)
c = UspCase(seq=L, hc=32, kv_hc=8, hs=128, ulysses=U, ring=R, causal=True)
g = torch.Generator(device=dev).manual_seed(1)
q = torch.randn(1, L, 32, 128, device=dev, dtype=torch.bfloat16, generator=g)
k = torch.randn(1, L, 8, 128, device=dev, dtype=torch.bfloat16, generator=g)
v = torch.randn(1, L, 8, 128, device=dev, dtype=torch.bfloat16, generator=g)
run_usp_gpu(c, q, k, v, dev)
torch.cuda.synchronize()
print("done")
