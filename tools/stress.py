"""Determinism / race stress: the same forward (and backward) many times,
outputs compared with the first run (development aid).
python tools/stress.py [iters]

The forward, and the backward in its deterministic (two-kernel) mode, must
be bit-identical run to run. The default fused backward reduces dQ partials
in arrival order: its dK / dV must still be bit-identical, its dQ within
fp32 reduction-order noise (max |diff| <= 1e-2 max|dQ|, typically a few
bf16 ulps on isolated elements); any larger difference is a race."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2405_07719_b200 import ProcessMesh, UspAttention  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
dev = torch.device("cuda", 0)


def same_grads(got, ref, det):
    """mismatch count: dk, dv (and dq when deterministic) bitwise; dq within noise otherwise"""
    bad = 0 if all(torch.equal(a, b) for a, b in zip(got[1:], ref[1:])) else 1
    if det:
        bad += 0 if torch.equal(got[0], ref[0]) else 1
    else:
        scale = float(ref[0].float().abs().max())
        bad += 0 if float((got[0].float() - ref[0].float()).abs().max()) <= 1e-2 * scale else 1
    return bad


for det in (False, True):
    for (L, hc, kv, hs, bwd) in ((2048, 32, 8, 128, True), (32768, 32, 8, 128, False), (4096, 8, 8, 64, True),
                                 (3000, 12, 4, 128, True), (2900, 8, 2, 128, True), (16384, 32, 8, 128, True)):
        if det and not bwd:
            continue
        eng = UspAttention(ProcessMesh(1, 1), rank=0, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True)
        eng.set_deterministic(det)
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
                bad += same_grads([gr.dq, gr.dk, gr.dv], rg, det)
        torch.cuda.synchronize()
        print(f"L={L} hc={hc} kv={kv} hs={hs} bwd={bwd} det={det}: {n} iterations, mismatches={bad}", flush=True)
        assert bad == 0

# multi-rank: in-process meshes (the Ulysses exchange pipelined in row chunks
# by default), forward + backward, many times
from tests.usp_harness import UspCase, run_usp_gpu_fwd_bwd  # noqa: E402

for (U, R) in ((2, 4), (4, 1), (2, 2)):
    for det in (False, True):
        c = UspCase(seq=4096, hc=32, kv_hc=8, hs=128, ulysses=U, ring=R, causal=True)
        g = torch.Generator(device=dev).manual_seed(7)
        q = torch.randn(1, c.seq, c.hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
        k = torch.randn(1, c.seq, c.kv_hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
        v = torch.randn(1, c.seq, c.kv_hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
        do = torch.randn(1, c.seq, c.hc, c.hs, device=dev, dtype=torch.bfloat16, generator=g)
        ref = [x.clone() for x in run_usp_gpu_fwd_bwd(c, q, k, v, do, dev, deterministic=det)[:4]]
        bad = 0
        n = max(10, iters // 10)
        for i in range(n):
            got = run_usp_gpu_fwd_bwd(c, q, k, v, do, dev, deterministic=det)[:4]
            bad += 0 if torch.equal(got[0], ref[0]) else 1
            bad += same_grads(got[1:], ref[1:], det)
        print(f"mesh U{U}R{R} L=4096 fwd+bwd det={det}: {n} iterations, mismatches={bad}", flush=True)
        assert bad == 0
