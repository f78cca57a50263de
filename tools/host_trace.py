"""Timeline of the host-buffer forward (USP_HOST_TRACE=1): python tools/host_trace.py [L]"""
import os, sys
os.environ["USP_HOST_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True)
pin = lambda shape, dt: torch.randn(shape, dtype=torch.float32).to(dt).pin_memory()  # noqa: E731
q, k, v = pin(eng.q_shape(), torch.bfloat16), pin(eng.kv_shape(), torch.bfloat16), pin(eng.kv_shape(), torch.bfloat16)
o = torch.empty(eng.q_shape(), dtype=torch.bfloat16).pin_memory()
lse = torch.empty(eng.lse_shape(), dtype=torch.float32).pin_memory()
for i in range(3):
    print("== call", i, file=sys.stderr)
    eng.forward_host(q, k, v, o, lse)
    torch.cuda.synchronize()
