"""Pipelined Ulysses all-to-alls: every member's T rows are
exchanged in row chunks, ring step 0 runs chunk c as soon as it has landed
and the last step sends chunk c's O rows while chunk c+1 computes
(usp_engine_set_a2a_chunks). The attention of a q row does not depend on how
the rows are chunked, so every chunk count must give bitwise-identical O and
LSE; the default (2 chunks) is also checked against the oracle, and the
executed collectives against the reference's ledger (one logical all-to-all
per tensor, as all_to_all_4d.cpp records it).

Runs on the in-process (local) transport: one GPU, one host thread per rank."""
import numpy as np
import pytest
import torch

from oracle.oracle import Oracle
from tests.usp_harness import LSE_TOL, O_REL_L2, O_TOL, UspCase, errors, make_globals, run_usp_gpu, to_bf16, widen

pytestmark = pytest.mark.gpu


def _run(c: UspCase, chunks, device):
    q, k, v = make_globals(c)
    tq, tk, tv = (to_bf16(x, device) for x in (q, k, v))

    def setup(engines):
        for e in engines:
            e.set_a2a_chunks(chunks)
            e.enable_timing(True)

    out, lses, engines, _ = run_usp_gpu(c, tq, tk, tv, device, setup=setup)
    torch.cuda.synchronize(device)
    stages = [e.stage_times() for e in engines]
    return (tq, tk, tv), out.clone(), [x.clone() for x in lses], engines, stages


@pytest.mark.parametrize("u,r", [(2, 1), (4, 1), (8, 1), (2, 2), (4, 2), (2, 4)])
def test_chunk_counts_bitwise_equal(cuda, u, r):
    c = UspCase(seq=4096, hc=32, kv_hc=8, hs=128, ulysses=u, ring=r, causal=True, seed=11 + u + r)
    base = None
    T = c.seq // (u * r)
    for chunks in (1, 2, 4):
        if T % (chunks * 128):
            continue
        (tq, tk, tv), out, lses, engines, stages = _run(c, chunks, cuda)
        assert all(e.a2a_chunks == chunks for e in engines)
        if base is None:
            base = (out, lses)
            qd, kd, vd = widen(tq), widen(tk), widen(tv)
            ref_out, ref_lse = Oracle.usp_forward(qd, kd, vd, c.ulysses, c.ring, c.causal)
            eo = errors(widen(out), ref_out)
            el = errors(np.stack([widen(x) for x in lses]), ref_lse)
            assert eo["max_abs"] <= O_TOL and eo["rel_l2"] <= O_REL_L2 and el["max_abs"] <= LSE_TOL, (eo, el)
        else:
            assert torch.equal(out, base[0]), (u, r, chunks)
            assert all(torch.equal(a, b) for a, b in zip(lses, base[1])), (u, r, chunks)
        names = {s["stage"] for s in stages[0]}
        if chunks > 1:
            # per-chunk stages: exposed wait for chunk c's rows, attention of
            # chunk c in step 0, the exchanges on the comm stream
            for ch in range(chunks):
                assert f"wait_in.{ch}" in names and f"attn0.{ch}" in names, names
                assert f"a2a_in.{ch}" in names and f"a2a_out.{ch}" in names, names
        # launches: pack + unpack + R steps, steps 0 and R-1 split in chunks
        split = (chunks - 1) * (1 if r == 1 else 2)
        assert all(r + 2 <= e.last_launches() <= r + 2 + split for e in engines), [e.last_launches() for e in engines]


def test_default_chunks_and_ledger(cuda):
    from paper_2405_07719_b200.usp import forward_ledger

    c = UspCase(seq=2048, hc=8, kv_hc=4, hs=128, ulysses=2, ring=2, causal=True, seed=5)
    (tq, tk, tv), out, lses, engines, _ = _run(c, 2, cuda)
    for e in engines:
        assert e.ledger() == forward_ledger(e.cfg), e.rank
    # eligibility: default 2 chunks at U > 1, bs = 1, whole tiles per chunk
    from paper_2405_07719_b200 import Comm, ProcessMesh, UspAttention

    mesh = ProcessMesh(2, 1)
    comm = Comm.local(2)
    ok = UspAttention(mesh, rank=0, seq_len=2048, heads=8, kv_heads=4, head_size=128, causal=True, comm=comm,
                      device=cuda.index or 0)
    assert ok.a2a_chunks == 2
    odd = UspAttention(mesh, rank=0, seq_len=384, heads=8, kv_heads=4, head_size=128, causal=True, comm=comm,
                       device=cuda.index or 0)
    assert odd.a2a_chunks == 1  # T = 192 rows: no whole-tile halves
    from paper_2405_07719_b200 import UspInvalidInput

    with pytest.raises(UspInvalidInput, match="whole query tiles"):
        odd.set_a2a_chunks(2)
    ok.close()
    odd.close()


@pytest.mark.parametrize("u,r,chunks,hs,causal", [(2, 1, 2, 128, True), (4, 1, 4, 128, True), (2, 2, 2, 128, True),
                                                   (4, 2, 2, 128, True), (2, 1, 1, 128, True), (2, 2, 2, 64, True),
                                                   (4, 1, 2, 128, False)])
def test_host_buffers_pipelined_bitwise(cuda, u, r, chunks, hs, causal):
    """usp_attn_fwd_host with chunked exchanges (engine.cu fwd_host_a2a):
    Q rows go up, are packed and exchanged per chunk, O rows are unpacked and
    go down per chunk — the same kernels and plans as the device-resident
    forward, so O and LSE must be bitwise equal to it (chunks = 1: the
    whole-shard copy path, as a control). Every rank calls from its own
    Python thread (ctypes releases the GIL), as the in-process world needs."""
    import threading

    c = UspCase(seq=4096, hc=32, kv_hc=8, hs=hs, ulysses=u, ring=r, causal=causal, seed=29 + u + r)
    q, k, v = make_globals(c)
    tq, tk, tv = (to_bf16(x, cuda) for x in (q, k, v))

    def setup(engines):
        for e in engines:
            e.set_a2a_chunks(chunks)

    out, lses, engines, _ = run_usp_gpu(c, tq, tk, tv, cuda, setup=setup)
    pos = [torch.tensor(e.positions(), dtype=torch.long, device=cuda) for e in engines]
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    hin = [(pin(tq[:, p]), pin(tk[:, p]), pin(tv[:, p])) for p in pos]
    hout = [(torch.full(tq[:, p].shape, float("nan"), dtype=torch.bfloat16).pin_memory(),
             torch.full(lses[i].shape, float("nan"), dtype=torch.float32).pin_memory()) for i, p in enumerate(pos)]
    errs = []

    def rank(i):
        try:
            for _ in range(2):  # the second call reuses staging buffers and events
                engines[i].forward_host(*hin[i], *hout[i])
            torch.cuda.synchronize(cuda)
        except Exception as e:  # noqa: BLE001
            errs.append(f"rank {i}: {e!r}")

    th = [threading.Thread(target=rank, args=(i,)) for i in range(len(engines))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs and not any(t.is_alive() for t in th), errs
    for i, p in enumerate(pos):
        oh, lh = hout[i]
        assert torch.equal(oh.view(torch.int16), out[:, p].cpu().view(torch.int16)), (i, chunks)
        assert torch.equal(lh.view(torch.int32), lses[i].cpu().view(torch.int32)), (i, chunks)
        assert engines[i].a2a_chunks == chunks
