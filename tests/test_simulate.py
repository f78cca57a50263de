"""The reference's public C ABI (uspsim_run, include/uspsim.h) served by the
B200 library (include/usp_sim.h, csrc/simulate.cu) — SURVEY §8(f) #2.

Pinned to reports of the reference's OWN uspsim_run (tests/golden/
simulate_golden.json, made by tests/golden/make_simulate_golden.py from
oracle/_ref/libuspsim_api.so):
  * every invalid-input report (ShardSpec / check_usp_inputs / cmd_simulate
    rejections, JSON type errors, bad envelopes, unknown commands) is
    byte-identical: status, JSON document (incl. the fnv1a config digest of
    the nlohmann-style dump), text, ledger CSV; these run without a GPU;
  * simulate reports (GPU): same envelope/digest, mesh, shape, seed, and the
    same collectives — every ledger CSV row of the reference except its
    position all_gathers, same (group, step, rank), bytes scaled from fp64 to
    bf16 elements (fp32 for the circulating dK/dV partials) — and the fp64
    check passes at the bf16 tolerance.
"""
import csv
import io
import json
import os

import pytest

from paper_2405_07719_b200 import sim
from paper_2405_07719_b200._lib import SIM_EXPORTS, lib

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "simulate_golden.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_exports_reference_abi():
    import re
    header = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "usp_sim.h")
    declared = set(re.findall(r"USP_API\s+[\w\s\*]+?\b(uspsim_\w+)\(", open(header).read()))
    assert declared == set(SIM_EXPORTS)
    L = lib()
    for name in SIM_EXPORTS:
        assert hasattr(L, name), name
    assert L.uspsim_version().decode().startswith("0.1.0")


@pytest.mark.parametrize("case", _golden()["invalid"], ids=lambda c: c["request"][:60])
def test_invalid_reports_identical_to_reference(case):
    ours = sim.run(case["request"])
    assert ours.status == case["status"]
    if case["json"] is None:  # no report: JSON parse failure, last error set
        assert ours.json is None
        assert ours.text.startswith("request is not valid JSON: ")
        return
    assert ours.json == case["json"]
    assert ours.text == case["text"]
    assert ours.ledger_csv == case["csv"] == ""


def test_bf16_is_the_only_precision():
    r = sim.run({"command": "simulate", "params": {"precision": "fp64"}})
    assert r.status == sim.USPSIM_INVALID_INPUT and r.exit_code == 2
    assert "precision must be \"bf16\"" in r.doc["results"]["error"]


def test_analytic_commands_are_rejected_with_a_pointer():
    for cmd in ("cost", "plan"):
        r = sim.run({"command": cmd, "params": {}})
        assert r.status == 2 and "not served by the B200 engine" in r.doc["results"]["error"]


def test_null_request():
    h = __import__("ctypes").c_void_p()
    assert lib().uspsim_run(None, __import__("ctypes").byref(h)) == 2
    assert lib().uspsim_last_error().decode() == "request_json is null"


# ---------------------------------------------------------------- GPU
def _rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def _expected_elem_bytes(ref_rows):
    """bytes per element each non-gather reference row moves on B200: bf16,
    except ring-group shifts after the group's backward all_gather that come
    in the dK/dV-partial slots (ring_attention.cpp:79-155: per step t, K and V
    while t < R-1, then dK and dV while t >= 1)."""
    out = {}
    by_group = {}
    for r in ref_rows:
        by_group.setdefault(r["group"], []).append(r)
    for g, rows in by_group.items():
        steps = sorted({int(r["step"]) for r in rows})
        kinds = {int(r["step"]): r["collective"] for r in rows}
        gathers = [s for s in steps if kinds[s] == "all_gather"]
        shifts_after = [s for s in steps if kinds[s] == "ring_shift" and len(gathers) > 1 and s > gathers[1]]
        n_ring = len(g.split(","))
        slots = []
        for t in range(n_ring):
            if t < n_ring - 1:
                slots += [2, 2]
            if t >= 1:
                slots += [4, 4]
        for s in steps:
            out[(g, s)] = 2
        for s, e in zip(shifts_after, slots):
            out[(g, s)] = e
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("case", _golden()["simulate"], ids=lambda c: c["request"][:80])
def test_simulate_matches_reference_report(cuda, case):
    ours = sim.run(case["request"])
    ref = json.loads(case["json"])
    doc = ours.doc
    assert ours.status == 0, ours.text
    for key in ("command", "config_digest", "params", "schema_version", "status", "exit_code"):
        assert doc[key] == ref[key], key
    res, rres = doc["results"], ref["results"]
    for key in ("world_size", "mesh", "shape", "causal", "seed"):
        assert res[key] == rres[key], key
    assert res["precision"] == "bf16"
    assert res["engine"]["kernel_launches"] >= 1
    if "check" in rres:
        c = res["check"]
        assert c["passed"] and max(c["max_abs_out"], c["max_abs_dq"], c["max_abs_dk"], c["max_abs_dv"]) <= \
            c["tolerance"] == 2e-2, c
    # ledger: every reference row except the position all_gathers
    ref_rows = [r for r in _rows(case["csv"]) if r["collective"] != "all_gather"]
    elem = _expected_elem_bytes(_rows(case["csv"]))
    our_rows = _rows(ours.ledger_csv)
    assert [(r["step"], r["collective"], r["group"], r["rank"]) for r in our_rows] == \
           [(r["step"], r["collective"], r["group"], r["rank"]) for r in ref_rows]
    hs = rres["shape"]["head_size"]
    pad = (64 if hs <= 64 else 128) / hs  # bytes as moved: head size zero-padded to the kernel's 64/128
    for o, r in zip(our_rows, ref_rows):
        assert float(o["bytes"]) == float(r["bytes"]) / 8 * elem[(r["group"], int(r["step"]))] * pad, (o, r)
    summ, rsumm = res["ledger"], rres["ledger"]
    assert summ["events_per_group"] == rsumm["events_per_group"]
    for kind, v in rsumm["collectives"].items():
        if kind == "all_gather":
            assert kind not in summ["collectives"]
        else:
            assert summ["collectives"][kind]["events"] == v["events"]


@pytest.mark.gpu
def test_simulate_c1_shape_checks(cuda):
    """configs[0]: L=4096, hc=8, hs=64, U2 x R2, causal, fwd+bwd, fp64 check."""
    r = sim.run({"command": "simulate", "params": {"seqlen": 4096, "heads": 8, "kv_heads": 8, "head_size": 64,
                                                   "ulysses": 2, "ring": 2, "causal": True, "check": True}})
    assert r.status == 0, r.text
    c = r.doc["results"]["check"]
    print(r.text, c)
    assert c["passed"] and c["max_abs_out"] < 5e-3


@pytest.mark.gpu
def test_simulate_tolerance_failure_is_exit_1(cuda):
    r = sim.run({"command": "simulate", "params": {"seqlen": 64, "heads": 4, "head_size": 16, "ring": 2,
                                                   "causal": True, "check": True, "tolerance": 1e-9}})
    assert r.status == sim.USPSIM_TOLERANCE_EXCEEDED and r.exit_code == 1
    assert r.doc["status"] == "tolerance_exceeded" and "FAIL" in r.text


@pytest.mark.parametrize("case", _golden()["balance"], ids=lambda c: c["request"][:60])
def test_balance_reports_identical_to_reference(case):
    """The `balance` command (commands.cpp:414-462): zigzag vs contiguous
    causal pair counts per ring rank, byte-identical to the reference."""
    ours = sim.run(case["request"])
    assert ours.status == case["status"]
    assert ours.json == case["json"]
    assert ours.text == case["text"]
