"""CPU tests of the native library's host logic through the C ABI (no GPU):
the library loads and exports every include/usp_attn.h symbol; layout,
validation and the per-step tile plans match the reference rules."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2405_07719_b200 import ProcessMesh, ShardSpec, UspInvalidInput, causal_pair_counts, zigzag_partition
from paper_2405_07719_b200._lib import EXPORTS, lib
from paper_2405_07719_b200.usp import make_config, rank_flops, schedule, step_plan

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "usp_attn.h")


def test_library_exports_every_declared_symbol():
    declared = set(re.findall(r"USP_API\s+[\w\s\*]+?\b(usp_\w+)\(", open(HEADER).read()))
    assert declared == set(EXPORTS)
    L = lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.usp_version().decode().startswith("0.1")


def test_zigzag_and_pair_counts_match_reference_rules():
    assert zigzag_partition(16, 4) == [[0, 1, 14, 15], [2, 3, 12, 13], [4, 5, 10, 11], [6, 7, 8, 9]]
    with pytest.raises(UspInvalidInput, match="not divisible by 2\\*ring"):
        zigzag_partition(10, 4)
    assert causal_pair_counts(zigzag_partition(16, 4), 16) == [34] * 4
    for L, R in ((4096, 8), (96, 3), (212992, 2)):
        assert np.array_equal(np.array(zigzag_partition(L, R)), Oracle.zigzag_partition(L, R))


@pytest.mark.parametrize("U,R,L,causal", [(2, 2, 8, True), (4, 2, 64, True), (2, 2, 8, False), (1, 8, 4096, True),
                                          (8, 1, 1024, False), (4, 2, 212992, True)])
def test_positions_match_oracle(U, R, L, causal):
    spec = ShardSpec(ProcessMesh(U, R), L, causal)
    for r in range(U * R):
        assert np.array_equal(spec.positions_for(r), Oracle.positions_for(U, R, L, causal, r))
    # gather_positions over the Ulysses group == concatenation of the members' positions
    mesh = ProcessMesh(U, R)
    for r in range(U * R):
        cat = sum((spec.positions_for(m) for m in mesh.ulysses_group(r)), [])
        assert spec.head_positions(r) == cat


def test_shard_spec_reference_example():
    spec = ShardSpec(ProcessMesh(2, 2), 8, True)  # test_usp.cpp:68-91
    assert [spec.positions_for(r) for r in range(4)] == [[0, 1], [6, 7], [2, 3], [4, 5]]


def test_validation_messages():
    from paper_2405_07719_b200.usp import UspConfig

    def validate(**kw):
        base = dict(ulysses_degree=1, ring_degree=1, rank=0, device=0, batch=1, seq_len=256, heads=32,
                    kv_heads=8, head_size=128, causal=1)
        base.update(kw)
        c = UspConfig(**base)
        st = lib().usp_config_validate(ctypes.byref(c))
        return st, lib().usp_last_error().decode()

    assert validate()[0] == 0
    st, msg = validate(ulysses_degree=16)
    assert st == 2 and "cannot exceed" in msg
    st, msg = validate(ring_degree=3, seq_len=100)
    assert st == 2 and "not divisible by 2*ring" in msg
    st, msg = validate(heads=30, kv_heads=8)
    assert st == 2 and "head count" in msg
    st, msg = validate(ulysses_degree=4, ring_degree=2, seq_len=8 * 2 + 4, causal=0)
    assert st == 2
    st, msg = validate(head_size=256)
    assert st == 2 and "128" in msg
    # 8-bit head field of the work units: > 256 local heads is rejected, not
    # silently aliased into the batch byte (round-1 advice)
    st, msg = validate(heads=512, kv_heads=8)
    assert st == 2 and "256 heads" in msg
    assert validate(heads=512, kv_heads=8, ulysses_degree=2)[0] == 0


@pytest.mark.parametrize("U,R,L", [(1, 1, 131072), (1, 8, 131072), (4, 2, 212992), (2, 4, 32768), (8, 1, 32768)])
def test_zigzag_balance_and_total_flops(U, R, L):
    hc, kv, hs = 32, 8, 128
    mesh = ProcessMesh(U, R)
    flops = [rank_flops(make_config(mesh, rank=r, seq_len=L, heads=hc, kv_heads=kv, head_size=hs, causal=True))
             for r in range(U * R)]
    total = 4 * hc * hs * L * (L + 1) / 2
    assert abs(sum(flops) - total) / total < 1e-12
    assert max(flops) == min(flops)  # zigzag: every rank does equal work


def _dense_mask(qp, kp, causal):
    return np.ones((len(qp), len(kp)), bool) if not causal else (np.asarray(kp)[None, :] <= np.asarray(qp)[:, None])


@pytest.mark.parametrize("U,R,L,causal", [(1, 1, 1000, True), (1, 4, 1024, True), (2, 2, 640, True),
                                          (1, 2, 512, False), (4, 2, 2048, True), (1, 3, 600, True)])
def test_tile_plan_covers_exactly_the_visible_pairs(U, R, L, causal):
    """Every (q tile, k tile) with a visible pair is in the plan; 'full'
    tiles are entirely visible; skipped tiles are entirely masked."""
    mesh = ProcessMesh(U, R)
    spec = ShardSpec(mesh, L, causal)
    for rank in range(U * R):
        cfg = make_config(mesh, rank=rank, seq_len=L, heads=U * 2, kv_heads=U, head_size=128, causal=causal)
        mine = spec.head_positions(rank)
        u, r = mesh.ulysses_coord(rank), mesh.ring_coord(rank)
        total_pairs = 0
        for step in range(R):
            info = schedule(cfg, step)
            src = (r - step + R) % R
            assert info.src_ring_coord == src
            assert info.send_to_rank == mesh.rank_of(u, (r + 1) % R)
            assert info.recv_from_rank == mesh.rank_of(u, (r - 1 + R) % R)
            kp = spec.head_positions(mesh.rank_of(u, src))
            mask = _dense_mask(mine, kp, causal)
            assert info.visible_pairs == mask.sum()
            total_pairs += info.visible_pairs
            off, lst = step_plan(cfg, step)
            nq = (len(mine) + 127) // 128
            nk = (len(kp) + 127) // 128
            planned = {}
            for qt in range(nq):
                for e in lst[off[qt]:off[qt + 1]]:
                    planned[(qt, int(e) & 0x7FFFFFFF)] = bool(int(e) & 0x80000000)
            for qt in range(nq):
                for kt in range(nk):
                    blk = mask[qt * 128:(qt + 1) * 128, kt * 128:(kt + 1) * 128]
                    ragged = blk.shape != (128, 128) and kt * 128 + 128 > len(kp)
                    if (qt, kt) not in planned:
                        assert not blk.any(), (rank, step, qt, kt)
                    elif not planned[(qt, kt)]:
                        assert blk.all() and not ragged, (rank, step, qt, kt)
        if causal:
            assert total_pairs == L * (L + 1) // 2 // R  # partition.cpp:52-72, zigzag-exact


def test_ring_bytes_per_step():
    # ledger closed form (ledger.cpp:34): ring shift bytes = buffer bytes per step, R-1 steps
    mesh = ProcessMesh(2, 4)
    cfg = make_config(mesh, rank=3, seq_len=4096, heads=32, kv_heads=8, head_size=128, causal=True)
    per_step = 2 * (4096 // 4) * (8 // 2) * 128 * 2  # K+V (L/R, kv/U, hs) bf16
    sent = [schedule(cfg, t).ring_bytes_sent for t in range(4)]
    assert sent == [per_step] * 3 + [0]
