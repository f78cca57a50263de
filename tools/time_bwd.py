"""Device timing of the U=R=1 backward (development aid).

Algorithmic FLOPs of the backward = 2.5x the forward's (five GEMMs of
2*hs per visible pair and head: S, dP, dV, dK, dQ); the two-kernel design
recomputes S and dP once more (7 GEMMs executed)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402


def run(L, hc=32, kv=8, hs=128, causal=True, iters=None, det=False):
    iters = iters or max(3, int(1e11 / (L * L)))
    dev = torch.device("cuda", 0)
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=causal)
    eng.set_deterministic(det)
    q = torch.randn(1, L, hc, hs, device=dev, dtype=torch.bfloat16)
    k = torch.randn(1, L, kv, hs, device=dev, dtype=torch.bfloat16)
    v = torch.randn(1, L, kv, hs, device=dev, dtype=torch.bfloat16)
    do = torch.randn(1, L, hc, hs, device=dev, dtype=torch.bfloat16)
    fwd = eng.forward(q, k, v)
    dq, dk, dv = eng.alloc_grads()
    for _ in range(2):
        eng.backward(fwd, do, dq, dk, dv)
    torch.cuda.synchronize()
    eng.enable_timing(True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.25)
    s.record()
    for _ in range(iters):
        eng.backward(fwd, do, dq, dk, dv)
    e.record()
    torch.cuda.synchronize()
    c = clk.stop()
    kt = eng.kernel_times()  # per iteration: fused | dkdv, dq
    eng.enable_timing(False)
    ms = s.elapsed_time(e) / iters
    fl = 2.5 * eng.flops()
    tf = fl / ms / 1e9
    F = eng.flops()  # forward: 2 GEMMs
    if len(kt) == iters:  # fused: 5 GEMMs executed = algorithmic
        fk = sum(kt) / iters
        detail = f"fused {fk:.3f} ms ({2.5 * F / fk / 1e9:.0f} TF/s)"
    else:
        dkdv = sum(kt[0::2]) / iters
        dqk = sum(kt[1::2]) / iters
        detail = (f"dkdv {dkdv:.3f} ms ({2 * F / dkdv / 1e9:.0f} TF/s executed) dq {dqk:.3f} ms "
                  f"({1.5 * F / dqk / 1e9:.0f})")
    print(f"bwd{' det' if det else ''} L={L} hc={hc} kv={kv} hs={hs} causal={causal}: {ms:.3f} ms  "
          f"{tf:.1f} TFLOP/s algorithmic | {detail} sm_mhz={c['sm_mhz']} {c['reasons']}", flush=True)
    eng.close()


if __name__ == "__main__":
    det = os.environ.get("BWD_DET") == "1"
    for L in [int(x) for x in (sys.argv[1:] or ["8192", "32768", "131072"])]:
        run(L, det=det)
