"""ncu target: one cuDNN SDPA forward (torch SDPBackend.CUDNN_ATTENTION) at the
bench head shape, for comparing its launch configuration and pipe use with
the repo's kernel (tools/ceiling.py has the timings).  python tools/profile_cudnn.py [L]"""
import sys

import torch
from torch.nn.attention import SDPBackend, sdpa_kernel

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
dev = torch.device("cuda", 0)
u = lambda *s: (torch.rand(s, device=dev) * 2 - 1).to(torch.bfloat16)  # noqa: E731
q, k, v = u(1, 32, L, 128), u(1, 8, L, 128), u(1, 8, L, 128)
with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
    for _ in range(2):
        torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
torch.cuda.synchronize()
