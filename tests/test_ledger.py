"""Comm-ledger parity: the collectives one rank's forward
issues, in the reference CommLedger's terms (src/simcomm/ledger.hpp:21-30,
closed forms ledger.cpp:25-37), against the ledger the reference's own
World recorded for the same forward (tests/golden, from oracle/_ref).

The reference additionally all_gathers the token positions twice per
forward (usp_attention.cpp:53, ring_attention.cpp:56); the B200 engine
computes that static layout on the host, so those two events are absent."""
import json
import os

import numpy as np
import pytest

from paper_2405_07719_b200 import ProcessMesh
from paper_2405_07719_b200.usp import backward_ledger, forward_ledger, make_config

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")
REF_ELEM = 8  # the golden forwards ran usp_attention<double>
OUR_ELEM = 2  # bf16


def _cases():
    g = np.load(GOLDEN)
    return [(k.split("/")[0], g[k.split("/")[0] + "/meta"], json.loads(str(g[k])))
            for k in g.files if k.endswith("/ledger")]


@pytest.mark.parametrize("name,meta,ref", _cases(), ids=lambda x: x if isinstance(x, str) else "")
def test_forward_ledger_matches_reference(name, meta, ref):
    bs, seq, hc, kv, hs, U, R, causal, _ = [int(x) for x in meta]
    mesh = ProcessMesh(U, R)
    ref_ev = [e for e in ref if e["kind"] != "all_gather"]
    ours = []
    for rank in range(U * R):
        cfg = make_config(mesh, rank=rank, seq_len=seq, heads=hc, kv_heads=kv, head_size=hs, causal=bool(causal),
                          batch=bs)
        for e in forward_ledger(cfg):
            members = [e["group_first"] + i * e["group_stride"] for i in range(e["group_size"])]
            ours.append((e["kind"], ",".join(map(str, members)), e["step"], e["payload_elems"],
                         e["bytes_sent"] / OUR_ELEM, rank))
    kinds = {3: "all_to_all", 4: "ring_shift"}
    # per group: same sequence of events (kind, payload), same bytes per member
    for grp in sorted({e["group"] for e in ref_ev}):
        r_seq = sorted((e for e in ref_ev if e["group"] == grp), key=lambda e: e["step"])
        members = [int(x) for x in grp.split(",")]
        for m_i, m in enumerate(members):
            o_seq = sorted((o for o in ours if o[1] == grp and o[5] == m), key=lambda o: o[2])
            assert [kinds[o[0]] for o in o_seq] == [e["kind"] for e in r_seq], (name, grp, m)
            assert [o[3] for o in o_seq] == [e["payload_elems"] for e in r_seq], (name, grp, m)
            assert [o[4] for o in o_seq] == [e["bytes_sent"][m_i] / REF_ELEM for e in r_seq], (name, grp, m)
    # nothing extra on our side
    assert len({(o[1], o[0], o[2]) for o in ours}) == len(ref_ev)


def test_closed_forms_gqa_u2r2():
    # test_usp.cpp:381-433 (forward half): 4 all-to-alls per Ulysses group,
    # K/V bytes = kv/hc x Q bytes, O bytes = Q bytes, 2(R-1) shifts per ring group
    mesh = ProcessMesh(2, 2)
    cfg = make_config(mesh, rank=1, seq_len=16, heads=8, kv_heads=2, head_size=4, causal=True, batch=2)
    ev = forward_ledger(cfg)
    a2a = [e for e in ev if e["kind"] == 3]
    shifts = [e for e in ev if e["kind"] == 4]
    assert len(a2a) == 4 and len(shifts) == 2 * (2 - 1)
    q, k, v, o = (e["bytes_sent"] for e in a2a)
    assert k == q * 2 / 8 and v == q * 2 / 8 and o == q


def _bwd_cases():
    g = np.load(GOLDEN)
    return [(k.split("/")[0], g[k.split("/")[0] + "/meta"], json.loads(str(g[k])))
            for k in g.files if k.endswith("/bwd_ledger")]


@pytest.mark.parametrize("name,meta,ref", _bwd_cases(), ids=lambda x: x if isinstance(x, str) else "")
def test_backward_ledger_matches_reference(name, meta, ref):
    """Forward + backward collectives (usp_attention.cpp:68-89,
    ring_attention.cpp:79-155) vs the reference World's ledger; the circulating
    dK/dV partials travel in fp32 (4 bytes), everything else in bf16."""
    bs, seq, hc, kv, hs, U, R, causal, _ = [int(x) for x in meta]
    mesh = ProcessMesh(U, R)
    ref_ev = [e for e in ref if e["kind"] != "all_gather"]
    kinds = {3: "all_to_all", 4: "ring_shift"}
    ours = []
    for rank in range(U * R):
        cfg = make_config(mesh, rank=rank, seq_len=seq, heads=hc, kv_heads=kv, head_size=hs, causal=bool(causal),
                          batch=bs)
        for e in backward_ledger(cfg):
            members = [e["group_first"] + i * e["group_stride"] for i in range(e["group_size"])]
            elem = 4 if e["tensor"] in (6, 7) and e["kind"] == 4 else OUR_ELEM
            ours.append((e["kind"], ",".join(map(str, members)), e["step"], e["payload_elems"],
                         e["bytes_sent"] / elem, rank))
    for grp in sorted({e["group"] for e in ref_ev}):
        r_seq = sorted((e for e in ref_ev if e["group"] == grp), key=lambda e: e["step"])
        for m_i, m in enumerate(int(x) for x in grp.split(",")):
            o_seq = sorted((o for o in ours if o[1] == grp and o[5] == m), key=lambda o: o[2])
            assert [kinds[o[0]] for o in o_seq] == [e["kind"] for e in r_seq], (name, grp, m)
            assert [o[3] for o in o_seq] == [e["payload_elems"] for e in r_seq], (name, grp, m)
            assert [o[4] for o in o_seq] == [e["bytes_sent"][m_i] / REF_ELEM for e in r_seq], (name, grp, m)
    assert len({(o[1], o[0], o[2]) for o in ours}) == len(ref_ev)
