"""Multi-process (gloo, CPU) test of the N>1 host path.

Each process is one rank of a U x R mesh. It takes its shard from the
library's ShardSpec (positions_for), then executes the engine's schedule
exactly as usp_attn_fwd does, with gloo send/recv standing in for NCCL and
the fp64 oracle standing in for the tcgen05 block kernel:
  1. Ulysses all-to-all in   (part p = heads [p*H/U, (p+1)*H/U), received
                              parts concatenated along seq in member order,
                              all_to_all_4d.cpp:13-59)
  2. R ring steps            (usp_schedule: source block, send/recv peers;
                              per-step LSE merge First/Middle/Last as the
                              kernel epilogue does)
  3. Ulysses all-to-all out  (all_to_all_4d.cpp:62-107)
and checks its O shard and head-sharded LSE against the single-device
oracle. This validates the host-side schedule, peers and layouts on
world_size 2 and 4 without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _a2a(parts, group_members, rank, tag):
    """all_to_all over a group with point-to-point gloo ops."""
    me = group_members.index(rank)
    recv = [None] * len(parts)
    reqs = []
    for p, peer in enumerate(group_members):
        if peer == rank:
            recv[p] = parts[p].copy()
            continue
        buf = torch.empty(parts[me].shape, dtype=torch.float64)
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(parts[p])), peer, tag=tag))
        reqs.append(dist.irecv(buf, peer, tag=tag))
        recv[p] = buf
    for r in reqs:
        r.wait()
    return [x if isinstance(x, np.ndarray) else x.numpy() for x in recv]


def _worker(rank, world, U, R, causal, port, errq):
    try:
        os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from oracle.oracle import Oracle
        from paper_2405_07719_b200 import ProcessMesh, ShardSpec
        from paper_2405_07719_b200.usp import make_config, schedule
        from tests.usp_harness import UspCase, make_globals

        c = UspCase(bs=1, seq=64 * U * R, hc=4 * U, kv_hc=2 * U, hs=8, ulysses=U, ring=R, causal=causal, seed=31)
        q, k, v = make_globals(c)
        mesh = ProcessMesh(U, R)
        spec = ShardSpec(mesh, c.seq, causal)
        cfg = make_config(mesh, rank=rank, seq_len=c.seq, heads=c.hc, kv_heads=c.kv_hc, head_size=c.hs,
                          causal=causal)
        pos = spec.positions_for(rank)
        qs, ks, vs = q[:, pos], k[:, pos], v[:, pos]
        hl, kvl = c.hc // U, c.kv_hc // U
        ug, rg = mesh.ulysses_group(rank), mesh.ring_group(rank)

        # 1. Ulysses in
        def heads_to_seq(x, local, tag):
            parts = [x[:, :, p * local:(p + 1) * local] for p in range(U)]
            return np.concatenate(_a2a(parts, ug, rank, tag), axis=1)

        qh, kh, vh = heads_to_seq(qs, hl, 1), heads_to_seq(ks, kvl, 2), heads_to_seq(vs, kvl, 3)
        head_pos = np.array(spec.head_positions(rank))
        assert np.array_equal(head_pos, np.concatenate([spec.positions_for(m) for m in ug]))

        # 2. ring
        o_run = lse_run = None
        k_cur, v_cur = kh, vh
        for step in range(R):
            info = schedule(cfg, step)
            src_rank = mesh.rank_of(mesh.ulysses_coord(rank), info.src_ring_coord)
            k_pos = np.array(spec.head_positions(src_rank))
            o_t, lse_t = Oracle.softmax_rows(qh, k_cur, v_cur, causal, head_pos, k_pos)
            o_t = np.nan_to_num(o_t)
            if o_run is None:  # EpiMode::kFirst / kSingle
                o_run, lse_run = o_t, lse_t
            else:  # kMiddle / kLast: log-sum-exp merge
                new = np.logaddexp(lse_run, lse_t)
                wa = np.where(np.isfinite(new), np.exp(lse_run - new), 0.0)[..., None]
                wb = np.where(np.isfinite(new), np.exp(lse_t - new), 0.0)[..., None]
                o_run, lse_run = o_run * wa + o_t * wb, new
            if step + 1 < R:
                bufk = torch.empty(k_cur.shape, dtype=torch.float64)
                bufv = torch.empty(v_cur.shape, dtype=torch.float64)
                reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(k_cur)), info.send_to_rank, tag=10 + step),
                        dist.isend(torch.from_numpy(np.ascontiguousarray(v_cur)), info.send_to_rank, tag=50 + step),
                        dist.irecv(bufk, info.recv_from_rank, tag=10 + step),
                        dist.irecv(bufv, info.recv_from_rank, tag=50 + step)]
                for r_ in reqs:
                    r_.wait()
                k_cur, v_cur = bufk.numpy(), bufv.numpy()
                assert rg[(rg.index(rank) + 1) % R] == info.send_to_rank

        # 3. Ulysses out
        T = len(pos)
        parts = [o_run[:, p * T:(p + 1) * T] for p in range(U)]
        out = np.concatenate(_a2a(parts, ug, rank, 99), axis=2)

        ref = Oracle.reference_attention(q, k, v, causal)
        err = np.abs(out - ref[:, pos]).max()
        _, ref_lse = Oracle.softmax_rows(q[:, head_pos][:, :, mesh.ulysses_coord(rank) * hl:][:, :, :hl],
                                         k[:, :, (mesh.ulysses_coord(rank) * kvl):][:, :, :kvl],
                                         v[:, :, (mesh.ulysses_coord(rank) * kvl):][:, :, :kvl],
                                         causal, head_pos, np.arange(c.seq))
        err_l = np.abs(lse_run - ref_lse).max()
        assert err < 1e-12 and err_l < 1e-12, (rank, err, err_l)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("U,R,causal", [(1, 2, True), (2, 1, True), (2, 1, False), (2, 2, True), (1, 4, True),
                                        (4, 1, False), (1, 2, False)])
def test_multi_process_schedule_gloo(U, R, causal):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    world = U * R
    procs = [ctx.Process(target=_worker, args=(r, world, U, R, causal, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs) and not errs, "\n".join(errs)
