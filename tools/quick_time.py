"""Quick device timing of the U=R=1 engine (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_07719_b200 import ProcessMesh, UspAttention
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler

def run(L, hc=32, kv=8, hs=128, causal=True, iters=None):
    iters = iters or max(5, int(4e11 / (L * L)))
    dev = torch.device("cuda", 0)
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=causal)
    q = torch.randn(1, L, hc, hs, device=dev, dtype=torch.bfloat16)
    k = torch.randn(1, L, kv, hs, device=dev, dtype=torch.bfloat16)
    v = torch.randn(1, L, kv, hs, device=dev, dtype=torch.bfloat16)
    o, lse = eng.alloc_outputs()
    for _ in range(2): eng.forward(q, k, v, o, lse)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(0); clk.start(); time.sleep(0.25)
    s.record()
    for _ in range(iters): eng.forward(q, k, v, o, lse)
    e.record(); torch.cuda.synchronize()
    c = clk.stop()
    ms = s.elapsed_time(e) / iters
    tf = eng.flops() / ms / 1e9
    print(f"L={L} hc={hc} kv={kv} hs={hs} causal={causal}: {ms:.3f} ms  {tf:.1f} TFLOP/s  ({tf/1640.5*100:.1f}% of 1640.5)  sm_mhz={c['sm_mhz']} {c['reasons']} W={c['power_w_max']}", flush=True)

if __name__ == "__main__":
    for L in [int(x) for x in (sys.argv[1:] or ["8192", "32768", "131072"])]:
        run(L)
    if len(sys.argv) == 1:
        run(32768, causal=False)
        run(8192, hc=8, kv=8, hs=64)
