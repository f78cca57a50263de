"""Determinism / race stress: the same forward (and backward) many times,
outputs compared bit for bit with the first run (development aid).
python tools/stress.py [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
dev = torch.device("cuda", 0)
for (L, hc, kv, hs, bwd) in ((2048, 32, 8, 128, True), (32768, 32, 8, 128, False), (4096, 8, 8, 64, True),
                             (3000, 12, 4, 128, True), (2900, 8, 2, 128, True)):
    eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True)
    g = torch.Generator(device=dev).manual_seed(L)
    q = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(eng.kv_shape(), device=dev, dtype=torch.bfloat16, generator=g)
    do = torch.randn(eng.q_shape(), device=dev, dtype=torch.bfloat16, generator=g)
    ref = eng.forward(q, k, v)
    ro, rl = ref.out.clone(), ref.logsumexp.clone()
    if bwd:
        g0 = eng.backward(ref, do)
        rg = [g0.dq.clone(), g0.dk.clone(), g0.dv.clone()]
    bad = 0
    n = iters if L <= 4096 else max(20, iters // 10)
    for i in range(n):
        f = eng.forward(q, k, v)
        if not (torch.equal(f.out, ro) and torch.equal(f.logsumexp, rl)):
            bad += 1
        if bwd:
            gr = eng.backward(f, do)
            if not all(torch.equal(a, b) for a, b in zip((gr.dq, gr.dk, gr.dv), rg)):
                bad += 1
    torch.cuda.synchronize()
    print(f"L={L} hc={hc} kv={kv} hs={hs} bwd={bwd}: {n} iterations, mismatches={bad}", flush=True)
    assert bad == 0

# multi-rank: a U2 x R4 in-process mesh, forward + backward, many times
from tests.usp_harness import UspCase, run_usp_gpu_fwd_bwd  # noqa: E402

c = UspCase(seq=4096, hc=32, kv_hc=8, hs=128, ulysses=2, ring=4, causal=True)
g = torch.Generator(device=dev).manual_seed(7)
q = torch.randn(1, c.seq, c.hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
k = torch.randn(1, c.seq, c.kv_hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
v = torch.randn(1, c.seq, c.kv_hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
do = torch.randn(1, c.seq, c.hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
ref = run_usp_gpu_fwd_bwd(c, q, k, v, do, dev)[:4]
ref = [x.clone() for x in ref]
bad = 0
n = max(10, iters // 10)
for i in range(n):
    got = run_usp_gpu_fwd_bwd(c, q, k, v, do, dev)[:4]
    bad += sum(0 if torch.equal(a, b) else 1 for a, b in zip(got, ref))
print(f"mesh U2R4 L=4096 fwd+bwd: {n} iterations, mismatches={bad}", flush=True)
assert bad == 0
