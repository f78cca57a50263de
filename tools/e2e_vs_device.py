"""Alternating device-resident vs host-buffer forwards, same power state (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=32, kv_heads=8, head_size=128, causal=True)
dev = torch.device("cuda", 0)
pin = lambda shape, dt: torch.randn(shape, dtype=torch.float32).to(dt).pin_memory()  # noqa: E731
qh, kh, vh = pin(eng.q_shape(), torch.bfloat16), pin(eng.kv_shape(), torch.bfloat16), pin(eng.kv_shape(), torch.bfloat16)
oh = torch.empty(eng.q_shape(), dtype=torch.bfloat16).pin_memory()
lh = torch.empty(eng.lse_shape(), dtype=torch.float32).pin_memory()
q, k, v = qh.to(dev), kh.to(dev), vh.to(dev)
o, lse = eng.alloc_outputs()
eng.forward(q, k, v, o, lse)
eng.forward_host(qh, kh, vh, oh, lh)
torch.cuda.synchronize()
for rnd in range(2):
    for mode in ("device", "host"):
        clk = ClockSampler(0)
        clk.start()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(4):
            if mode == "device":
                eng.forward(q, k, v, o, lse)
            else:
                eng.forward_host(qh, kh, vh, oh, lh)
        e.record()
        torch.cuda.synchronize()
        c = clk.stop()
        print(f"{mode}: {s.elapsed_time(e) / 4:.2f} ms/forward  sm_mhz={c['sm_mhz']}", flush=True)
