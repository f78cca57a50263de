"""Does concurrent PCIe traffic slow the attention kernel? (development aid)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402

L = 131072
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True)
dev = torch.device("cuda", 0)
q = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16)
k = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
v = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16)
o, lse = eng.alloc_outputs()
hu = torch.empty(1600 << 20, dtype=torch.uint8).pin_memory()
hd = torch.empty(1100 << 20, dtype=torch.uint8).pin_memory()
du = torch.empty(1600 << 20, dtype=torch.uint8, device=dev)
dd = torch.empty(1100 << 20, dtype=torch.uint8, device=dev)
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("alone", "with copies", "alone"):
    for _ in range(2):
        eng.forward(q, k, v, o, lse)
    torch.cuda.synchronize()
    clk = ClockSampler(0)
    clk.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(4):
        if mode == "with copies":
            with torch.cuda.stream(s_up):
                du.copy_(hu, non_blocking=True)
            with torch.cuda.stream(s_dn):
                hd.copy_(dd, non_blocking=True)
        eng.forward(q, k, v, o, lse)
    e.record()
    torch.cuda.synchronize()
    c = clk.stop()
    print(f"{mode}: {s.elapsed_time(e) / 4:.2f} ms/forward  sm_mhz={c['sm_mhz']} W={c['power_w_max']}", flush=True)
