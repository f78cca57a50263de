"""compute-sanitizer target (development aid): small U x R forward + backward
(fused and deterministic) at head sizes 128 and 64 on the in-process world.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from tests.usp_harness import UspCase, make_globals, make_globals_with_dout, run_usp_gpu_fwd_bwd, to_bf16
dev = torch.device("cuda", 0)
for (u, r, hs) in [(1, 1, 128), (2, 2, 128), (2, 1, 64)]:
    c = UspCase(seq=1024, hc=8, kv_hc=4, hs=hs, ulysses=u, ring=r, causal=True, seed=3)
    q, k, v, do = make_globals_with_dout(c)
    tq, tk, tv, tdo = (to_bf16(x, dev) for x in (q, k, v, do))
    for det in (False, True):
        out, dq, dk, dv, engines, comm = run_usp_gpu_fwd_bwd(c, tq, tk, tv, tdo, dev, deterministic=det)
        torch.cuda.synchronize()
        print("ok", u, r, hs, det, float(out.float().abs().mean()), float(dq.float().abs().mean()), flush=True)
        for e in engines: e.close()
