#!/usr/bin/env python
"""USP attention forward benchmark (the BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

One "step" = one USP attention forward (usp_attn_fwd through the C ABI) of
the Llama-3-8B attention layer (hc=32, kv=8, hs=128, bs=1) at L=128K,
causal with zigzag load balance, over a U x R mesh of N GPUs (default pure
ring, U=1, R=N: config c3; N=1 is the single-GPU kernel). Inputs are
synthetic: U[-1, 1) (the reference generator's range) drawn in
fp32 by a seeded torch generator on the GPU, rounded to bf16 and resident in
HBM; Q alone is 1 GiB, larger than the 126 MB L2, so no flush is needed
between steps. Prints ONE JSON line on rank 0.

Without WORLD_SIZE in the environment, --gpus N > 1 re-launches itself
under torch.distributed.run (N local ranks, 127.0.0.1).

Beside the throughput the line carries: `parity` (sampled query rows of the
timed forward against the fp64 oracle on the same bf16 inputs, and against
the reference's own fp32 SoftmaxState on the un-rounded inputs), `roofline`
(the attention kernel vs the bf16 tensor peak), `whole_forward` (SURVEY
§8(d)'s T_roof = A2A/BW + sum_t max(F_t/P, KV_t/BW) against the measured
forward), `stages_ms_per_step` (pack / a2a / per-ring-step attention / the
exposed part of each K/V shift / a2a out / unpack, CUDA events on the
forward's stream) and `cpu_baseline`.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libuspref.so: usp_attention<float> on U*R rank threads,
compiled from /root/reference sources) on a bounded sample of the same
workload, with as many host threads as its mesh allows.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "USP attn fwd TFLOP/s, L=128K Llama3-8B layer, 1/2/4/8 B200; % of BF16 peak"
UNIT = "TFLOP/s"


def self_launch_if_needed(a) -> bool:
    """--gpus N > 1 without a torch.distributed environment: run N local ranks
    under torch.distributed.run (the driver may call `python bench.py --gpus N`)."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ or a.impl == "reference":
        return False
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.run(cmd).returncode
    raise SystemExit(rc)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--head-size", type=int, default=128)
    ap.add_argument("--ulysses", type=int, default=1, help="Ulysses degree U (R = N / U)")
    ap.add_argument("--non-causal", action="store_true")
    ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl",
                    help="N>1 exchange: NCCL all-to-all + send/recv (north star), or the peer-memory "
                         "transport (CUDA IPC + copy engines, no SMs reserved)")
    ap.add_argument("--cpu-sample-len", type=int, default=4096)
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-backward", action="store_true")
    ap.add_argument("--backward-multi", action="store_true",
                    help="also report the backward when N > 1 (default: N = 1 only; the multi-GPU NCCL backward "
                         "has no one-GPU test, so the scaling runs do not depend on it)")
    ap.add_argument("--bwd-steps", type=int, default=3, help="timed steps of the backward report (both modes)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--parity-rows", type=int, default=12, help="sampled query rows checked vs the fp64 oracle")
    ap.add_argument("--parity-ref-rows", type=int, default=4,
                    help="sampled rows checked vs the reference's fp32 SoftmaxState")
    ap.add_argument("--skip-parity", action="store_true")
    return ap.parse_args()


def causal_flops(L, hc, hs, causal=True, batch=1):
    pairs = L * (L + 1) // 2 if causal else L * L
    return 4.0 * batch * hc * hs * pairs


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


def workload_config(a, n, U, R):
    return {
        **({"transport": a.transport} if n > 1 else {}),
        "workload": f"usp_attn_fwd llama3-8b layer L={a.seq_len} {'causal zigzag' if not a.non_causal else 'full'}",
        "seq_len": a.seq_len, "batch": 1, "heads": a.heads, "kv_heads": a.kv_heads, "head_size": a.head_size,
        "causal": not a.non_causal, "ulysses": U, "ring": R, "parallelism": f"u{U}r{R}",
        "l2": "inputs larger than L2 (Q alone %d MiB > 126 MB); no flush" % (a.seq_len * a.heads * a.head_size * 2 // n >> 20),
    }


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------- reference
def reference_mesh(kv_heads, seq_len, threads):
    """Largest U*R <= threads the reference accepts (U | kv, L % 2R == 0)."""
    best = (1, 1)
    for U in range(1, kv_heads + 1):
        if kv_heads % U:
            continue
        for R in range(1, threads // U + 1):
            if seq_len % (2 * R) or (seq_len // R) % U:
                continue
            if U * R > best[0] * best[1] or (U * R == best[0] * best[1] and U > best[0]):
                best = (U, R)
    return best


def cpu_reference_sample(a, repeats=1):
    """Times the reference CPU forward on one bounded sample; returns a dict."""
    import numpy as np

    from oracle.oracle import Oracle, Reference

    L, hc, kv, hs = a.cpu_sample_len, a.heads, a.kv_heads, a.head_size
    causal = not a.non_causal
    cores = os.cpu_count() or 1
    g = Oracle.uniform(0, L * hc * hs + 2 * L * kv * hs)
    q = g[:L * hc * hs].reshape(1, L, hc, hs)
    k = g[L * hc * hs:L * hc * hs + L * kv * hs].reshape(1, L, kv, hs)
    v = g[L * hc * hs + L * kv * hs:].reshape(1, L, kv, hs)
    f = causal_flops(L, hc, hs, causal)
    if Reference.available():
        U, R = reference_mesh(kv, L, cores)
        secs = [Reference.usp_forward(q, k, v, U, R, causal, precision="fp32", want_out=False)[2]
                for _ in range(repeats)]
        kind, threads = "reference", U * R
        sample = (f"reference usp_attention<float> (oracle/_ref, built from /root/reference sources), "
                  f"L={L} hc={hc} kv={kv} hs={hs} {'causal' if causal else 'full'}, mesh U{U}xR{R} = {U * R} "
                  f"rank threads of {cores} host cores; x{repeats}")
    else:
        secs = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            Oracle.usp_forward(q, k, v, 1, 1, causal)
            secs.append(time.perf_counter() - t0)
        kind, threads = "port", cores
        sample = (f"oracle C port (fp64, OpenMP) of the reference forward, L={L} hc={hc} kv={kv} hs={hs}; "
                  f"x{repeats}")
    mean = sum(secs) / len(secs)
    return {"value": f / mean / 1e12, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
            "seconds_per_sample": mean, "flops_per_sample": f,
            "extrapolated_full_workload_s": causal_flops(a.seq_len, hc, hs, causal) / (f / mean)}


def run_reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    n = a.gpus
    U = a.ulysses
    R = max(1, n // U)
    if rank != 0:
        return
    for _ in range(a.warmup):
        cpu_reference_sample(a)
    vals, secs = [], []
    for _ in range(a.steps):
        r = cpu_reference_sample(a)
        vals.append(r["value"])
        secs.append(r["seconds_per_sample"])
    v = sum(vals) / len(vals)
    cfg = workload_config(a, n, U, R)
    cfg["sample"] = r["sample"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": n, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1000 * sum(secs) / len(secs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["cores"], "kind": r["kind"], "sample": r["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours
def global_inputs(a, dev):
    """Global Q, K, V (fp32, U[-1, 1)) from one seeded stream in Q, K, V order
    (the reference fills Q, K, V from one UniformSource, commands.cpp:90-102)."""
    import torch

    gen = torch.Generator(device=dev).manual_seed(0)
    L = a.seq_len

    def draw(h):
        return torch.rand((1, L, h, a.head_size), device=dev, dtype=torch.float32, generator=gen).mul_(2).sub_(1)

    return draw(a.heads), draw(a.kv_heads), draw(a.kv_heads)


def parity_block(a, eng, g, out, lse, positions, U, rank_u):
    """Sampled rows of this rank's timed forward vs (i) the fp64 oracle on the
    same bf16 inputs and (ii) the reference's own fp32 SoftmaxState on the
    un-rounded fp32 inputs (commands.cpp:142-158)."""
    import numpy as np
    import torch

    from oracle.oracle import Oracle, Reference

    t0 = time.perf_counter()
    T = len(positions)
    hl = a.heads // U
    rng = np.random.default_rng(7)
    cand = [0, 1, T // 2 - 1, T // 2, T - 2, T - 1] + rng.integers(0, T, size=64).tolist()
    rows = sorted(set(cand))[: max(1, a.parity_rows)]
    rows = sorted(set([0, T - 1] + rows))[: max(2, a.parity_rows)]
    qpos = np.array([positions[i] for i in rows], np.int64)
    qf, kf, vf = g
    bf = lambda t: t.to(torch.bfloat16).double().cpu().numpy()  # noqa: E731
    q_rows_b = bf(qf[:, torch.tensor(qpos, device=qf.device)])
    kb, vb = bf(kf), bf(vf)
    kpos = np.arange(a.seq_len, dtype=np.int64)
    causal = not a.non_causal
    ref_o, ref_l = Oracle.softmax_rows(q_rows_b, kb, vb, causal, qpos, kpos)
    got_o = out[:, torch.tensor(rows, device=out.device)].double().cpu().numpy()
    hp = eng.head_positions()
    hidx = {p: i for i, p in enumerate(hp)}
    got_l = lse[:, torch.tensor([hidx[int(p)] for p in qpos], device=lse.device)].double().cpu().numpy()
    ref_l_loc = ref_l[:, :, rank_u * hl:(rank_u + 1) * hl]

    def errs(got, want):
        d = np.abs(got - want)
        return float(d.max()), float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))

    o_abs, o_rel = errs(got_o, ref_o)
    l_abs, _ = errs(got_l, ref_l_loc)
    tol = {"o_max_abs": 5e-3, "o_rel_l2": 3e-3, "lse_max_abs": 1e-4}
    blk = {"rows": len(rows), "heads": a.heads, "keys": a.seq_len,
           "oracle": "fp64 SoftmaxState restatement (oracle/usp_oracle.c, pinned bitwise to the reference) on "
                     "the same bf16-rounded inputs; O rows in positions_for order, LSE head-sharded",
           "o_max_abs": o_abs, "o_rel_l2": o_rel, "lse_max_abs": l_abs, "tol": tol,
           "pass": o_abs <= tol["o_max_abs"] and o_rel <= tol["o_rel_l2"] and l_abs <= tol["lse_max_abs"]}
    nref = min(a.parity_ref_rows, len(rows))
    if nref > 0 and Reference.available():
        import concurrent.futures as cf

        sel = np.linspace(0, len(rows) - 1, nref).astype(int)
        qf_rows = qf[:, torch.tensor(qpos[sel], device=qf.device)].double().cpu().numpy()
        kd, vd = kf.double().cpu().numpy(), vf.double().cpu().numpy()

        def one(j):
            return Reference.softmax_rows(qf_rows[:, j:j + 1], kd, vd, causal, qpos[sel][j:j + 1], kpos,
                                          precision="fp32")

        with cf.ThreadPoolExecutor(max_workers=nref) as ex:
            res = list(ex.map(one, range(nref)))
        r_o = np.concatenate([r[0] for r in res], axis=1)
        r_l = np.concatenate([r[1] for r in res], axis=1)[:, :, rank_u * hl:(rank_u + 1) * hl]
        fo_abs, fo_rel = errs(got_o[:, sel], r_o)
        fl_abs, _ = errs(got_l[:, sel], r_l)
        blk["vs_reference_fp32"] = {
            "rows": nref, "o_max_abs": fo_abs, "o_rel_l2": fo_rel, "lse_max_abs": fl_abs,
            "reference": "the reference's SoftmaxState<float>::update/finalize/logsumexp (oracle/_ref, built "
                         "from /root/reference sources) on the un-rounded fp32 inputs: the difference includes "
                         "the bf16 rounding of Q/K/V the GPU path takes"}
    blk["seconds"] = time.perf_counter() - t0
    return blk


def nccl_bandwidth(dev, world, U, R, rank, same_dev):
    """Measured NCCL bus bandwidth on this node for the two exchanges (GB/s of
    bytes sent per rank): all_to_all over the Ulysses rows and the ring
    send/recv over the columns, 64 MiB per rank, CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    if world == 1 or same_dev:
        return None
    out = {}
    nbytes = 64 << 20
    x = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # all_to_all over the whole world as a proxy for one Ulysses row (every
    # peer is one NVSwitch hop away)
    for _ in range(3):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize(dev)
    s0.record()
    for _ in range(5):
        dist.all_to_all_single(y, x)
    s1.record()
    torch.cuda.synchronize(dev)
    ms = s0.elapsed_time(s1) / 5
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["a2a_gbs"] = nbytes * (world - 1) / world / (t.item() * 1e-3) / 1e9
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    for it in range(8):
        if it == 3:
            torch.cuda.synchronize(dev)
            s0.record()
        ops = [dist.P2POp(dist.isend, x, nxt), dist.P2POp(dist.irecv, y, prv)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    s1.record()
    torch.cuda.synchronize(dev)
    ms = s0.elapsed_time(s1) / 5
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["p2p_gbs"] = nbytes / (t.item() * 1e-3) / 1e9
    out["kind"] = "measured: torch.distributed NCCL all_to_all_single / ring send-recv, 64 MiB per rank"
    return out


def whole_forward_roofline(eng, U, R, ms, peak, bw):
    """T_roof = A2A_bytes/BW_a2a + sum_t max(F_t/P, KV_t/BW_p2p)
    per rank; frac = T_roof / T_measured."""
    from paper_2405_07719_b200.usp import forward_ledger, schedule

    cfg = eng.cfg
    led = forward_ledger(cfg)
    a2a = sum(e["bytes_sent"] for e in led if e["kind"] == 3)
    nominal = 900.0
    bw_a2a = (bw or {}).get("a2a_gbs") or nominal
    bw_p2p = (bw or {}).get("p2p_gbs") or nominal
    hl = cfg.heads // U
    t = a2a / (bw_a2a * 1e9)
    terms, comm_bound = [], 0
    for st in range(R):
        info = schedule(cfg, st)
        f = 4.0 * cfg.batch * hl * cfg.head_size * info.visible_pairs
        tc = f / (peak * 1e12)
        tk = info.ring_bytes_sent / (bw_p2p * 1e9)
        terms.append(max(tc, tk))
        comm_bound += tk > tc
    t += sum(terms)
    return {"t_roof_ms": t * 1e3, "t_measured_ms": ms, "frac": (t * 1e3) / ms, "a2a_bytes_per_rank": a2a,
            "kv_bytes_per_shift": schedule(cfg, 0).ring_bytes_sent if R > 1 else 0,
            "bw_a2a_gbs": bw_a2a, "bw_p2p_gbs": bw_p2p,
            "bw_kind": (bw or {}).get("kind", "nominal NVLink 5 (900 GB/s per direction)") if U * R > 1 else "n/a",
            "peak_tflops": peak, "ring_steps_comm_bound": comm_bound,
            "a2a_ms": a2a / (bw_a2a * 1e9) * 1e3}


def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_2405_07719_b200 import Comm, ProcessMesh, UspAttention

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = a.gpus
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    # Development only: USP_BENCH_SAME_DEVICE=1 puts every rank on cuda:0
    # (gloo for the host plumbing, the p2p transport for the data) so the
    # multi-process path of this script can be exercised on a one-GPU box;
    # its numbers measure N processes sharing one GPU, not scaling.
    same_dev = os.environ.get("USP_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
        a.transport = "p2p"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1
    if distributed:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    U = a.ulysses
    if n % U:
        raise SystemExit("ulysses degree must divide the GPU count")
    R = n // U
    mesh = ProcessMesh(U, R)
    comm = None
    if distributed:
        if a.transport == "nccl":
            try:
                comm = Comm.from_torch_distributed(local)
            except Exception as e:  # every rank fails the same init the same way
                print(f"NCCL transport unavailable ({e}); using the peer-memory transport", file=sys.stderr)
                a.transport = "p2p (nccl init failed)"
        if comm is None:
            comm = Comm.p2p_from_torch_distributed(local)
    causal = not a.non_causal
    eng = UspAttention(mesh, rank=rank, seq_len=a.seq_len, heads=a.heads, kv_heads=a.kv_heads,
                       head_size=a.head_size, causal=causal, device=local, comm=comm)
    # global U[-1, 1) inputs (identical on every rank: same seed), this rank's
    # rows = ShardSpec::positions_for(rank) (zigzag when causal)
    positions = eng.positions()
    pos_t = torch.tensor(positions, dtype=torch.long, device=dev)
    g = global_inputs(a, dev)
    q, k, v = (x[:, pos_t].to(torch.bfloat16).contiguous() for x in g)
    if rank != 0 or a.skip_parity:
        del g
        g = None
    torch.cuda.empty_cache()
    o, lse = eng.alloc_outputs()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if distributed:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not distributed:
            return x
        t = torch.tensor([x], device="cpu" if same_dev else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(a.warmup):
        eng.forward(q, k, v, o, lse, stream)
    torch.cuda.synchronize(dev)

    # ---- timed region (device time, CUDA events, max over ranks)
    clocks = ClockSampler(local)
    launches = 0
    barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    eng.enable_timing(True)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(a.steps):
        eng.forward(q, k, v, o, lse, stream)
        launches += eng.last_launches()
    t1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / a.steps
    kts = eng.kernel_times()
    stages = {x["stage"]: x["ms_total"] / a.steps for x in eng.stage_times()}
    eng.enable_timing(False)
    ms = max_over_ranks(ms)

    rank_flops = eng.flops()
    total_flops = causal_flops(a.seq_len, a.heads, a.head_size, causal)
    value = total_flops / (ms * 1e-3) / 1e12
    peak, peak_sus, peak_kind = peaks()

    # roofline of the dominant kernel: algorithmic FLOPs per launch / mean
    # launch duration, both over the timed region
    kernel_ms = sum(kts) / len(kts) if kts else None
    flops_per_launch = rank_flops * a.steps / max(len(kts), 1)
    achieved = flops_per_launch / (kernel_ms * 1e-3) / 1e12 if kernel_ms else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tr = json.load(f)
            key = f"L{a.seq_len}_u{U}r{R}_{'causal' if causal else 'full'}"
            traffic = tr.get(key, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": UNIT,
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_kind": f"{peak_kind} burst bf16_tflops (cuBLAS)",
                "frac_of_sustained": (achieved / peak_sus) if achieved else None,
                "kernel_ms_mean": kernel_ms, "launches_timed": len(kts),
                "flops_per_launch": flops_per_launch}

    # ---- e2e through the public API: pinned host -> device, forward, device -> host
    e2e = None
    if not a.skip_e2e:
        qh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True).copy_(q)
        kh = torch.empty(k.shape, dtype=k.dtype, pin_memory=True).copy_(k)
        vh = torch.empty(v.shape, dtype=v.dtype, pin_memory=True).copy_(v)
        oh = torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
        lh = torch.empty(lse.shape, dtype=lse.dtype, pin_memory=True)

        def e2e_step():
            # host buffers in, host buffers out: the copies run inside the call
            eng.forward_host(qh, kh, vh, oh, lh, stream)

        e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1) / a.e2e_steps)
        h2d = sum(t.numel() * t.element_size() for t in (q, k, v))
        d2h = o.numel() * o.element_size() + lse.numel() * lse.element_size()
        e2e = {"value": total_flops / (ems * 1e-3) / 1e12, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems, "steps": a.e2e_steps,
               "path": "paper_2405_07719_b200.UspAttention.forward_host -> usp_attn_fwd_host (C ABI, pinned host "
                       "buffers; H2D/D2H pipelined against the attention in sequence chunks at U=R=1)"}

    # ---- backward of the same workload, reported beside
    # the forward metric: algorithmic FLOPs = 2.5 x the forward's (five
    # GEMM-equivalents of the forward's two), device time, max over ranks
    backward = None
    if not a.skip_backward and (not distributed or a.backward_multi):
        fwd = eng.forward(q, k, v, o, lse, stream)
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)
        dout = (torch.rand(q.shape, device=dev, generator=gen) * 2 - 1).to(torch.bfloat16)
        dq, dk, dv = eng.alloc_grads()
        backward = {"unit": UNIT, "flop_factor": 2.5, "steps": a.bwd_steps}
        for mode, det in (("fused", False), ("deterministic", True)):
            eng.set_deterministic(det)
            eng.backward(fwd, dout, dq, dk, dv, stream)  # warm-up (plans for this mode)
            torch.cuda.synchronize(dev)
            barrier()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            for _ in range(a.bwd_steps):
                eng.backward(fwd, dout, dq, dk, dv, stream)
            b1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
            bms = max_over_ranks(b0.elapsed_time(b1) / a.bwd_steps)
            backward[mode] = {"value": 2.5 * total_flops / (bms * 1e-3) / 1e12, "ms_per_step": bms,
                              "launches_per_step": eng.last_launches()}
        eng.set_deterministic(False)
        backward["value"] = backward["fused"]["value"]
        backward["kernel"] = ("fused: fa_bwd_fused_kernel (one launch per ring step, dQ TMA-reduced in fp32); "
                              "deterministic: fa_bwd_dkdv_kernel + fa_bwd_dq_kernel")
        del fwd, dout, dq, dk, dv

    bw = nccl_bandwidth(dev, world, U, R, rank, same_dev) if distributed else None
    whole = whole_forward_roofline(eng, U, R, ms, peak, bw)

    parity = None
    if rank == 0 and not a.skip_parity:
        try:
            parity = parity_block(a, eng, g, o, lse, positions, U, mesh.ulysses_coord(rank))
        except Exception as e:  # reported, not fatal
            parity = {"error": repr(e)}
    g = None

    cpu = None
    if rank == 0 and not a.skip_cpu_baseline:
        try:
            cpu = cpu_reference_sample(a, repeats=2)
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "unavailable", "sample": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic U[-1,1) (seeded torch generator, fp32 rounded to bf16), resident in HBM",
            "config": workload_config(a, n, U, R),
            "pct_of_peak_per_gpu": value / n / peak * 100.0,
            "tokens_per_s": a.seq_len / (ms * 1e-3),
            "roofline": roofline, "whole_forward": whole, "stages_ms_per_step": stages, "parity": parity,
            "cpu_baseline": cpu, "clocks": clk, "e2e": e2e, "backward": backward,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    self_launch_if_needed(a)
    if a.impl == "reference":
        run_reference_arm(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
