"""Collective failure diagnosis (CPU, no GPU work).

The reference World reports a mismatched collective ("collective mismatch on
group [g] call #k: rank a called X but rank b called Y", world.cpp:152-165)
and a world where every live rank is stuck ("collective deadlock: rank r
blocked at ...", world.cpp:89-113) instead of hanging. The local transport
keys its host rendezvous the same way (group, per-group call number,
signature) and bounds the wait by the comm timeout; once failed, every later
collective on the comm reports the failure (usp_comm_status too). Rank
threads here are Python threads calling the C ABI (ctypes releases the GIL),
as World::run runs one std::thread per rank.
"""
import threading

import pytest

from paper_2405_07719_b200 import Comm, UspError


def _run_ranks(fns):
    errs = [None] * len(fns)

    def wrap(i):
        try:
            fns[i]()
        except Exception as e:  # noqa: BLE001 - collected for the asserts
            errs[i] = e

    ts = [threading.Thread(target=wrap, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    assert not any(t.is_alive() for t in ts), "a rank hung"
    return errs


def test_matching_rendezvous_completes():
    c = Comm.local(2)
    c.set_timeout(5)
    sig = "all_to_all<bf16>(tensors=3,part_bytes=16/4/4)"
    errs = _run_ranks([lambda r=r: [c.debug_rendezvous(r, [0, 1], sig) for _ in range(3)] for r in range(2)])
    assert errs == [None, None]
    c.status()
    c.close()


def test_mismatched_collective_is_reported():
    c = Comm.local(2)
    c.set_timeout(5)
    a = "all_to_all<bf16>(tensors=3,part_bytes=16/4/4)"
    b = "ring_shift(buffers=2,bytes=64,steps=1)"
    errs = _run_ranks([lambda: c.debug_rendezvous(0, [0, 1], a), lambda: c.debug_rendezvous(1, [0, 1], b)])
    assert all(isinstance(e, UspError) and e.status == 3 for e in errs), errs
    msg = str(errs[0])
    assert "collective mismatch on group [0,1] call #0" in msg, msg
    assert "rank 0 called " + a in msg and "rank 1 called " + b in msg, msg
    with pytest.raises(UspError, match="collective mismatch"):
        c.status()
    with pytest.raises(UspError, match="collective mismatch"):  # the comm stays failed
        c.debug_rendezvous(0, [0, 1], a)
    c.close()


def test_missing_rank_is_reported_not_hung():
    c = Comm.local(3)
    c.set_timeout(1.0)
    sig = "ring_shift(buffers=2,bytes=64,steps=1)"
    # rank 2 never reaches its second ring shift; ranks 0 and 1 must report
    errs = _run_ranks([
        lambda: [c.debug_rendezvous(0, [0, 1, 2], sig) for _ in range(2)],
        lambda: [c.debug_rendezvous(1, [0, 1, 2], sig) for _ in range(2)],
        lambda: c.debug_rendezvous(2, [0, 1, 2], sig),
    ])
    assert errs[2] is None
    for e in errs[:2]:
        assert isinstance(e, UspError), errs
        assert "collective deadlock" in str(e), str(e)
        assert "blocked at " + sig + " call #1 on group [0,1,2]" in str(e), str(e)
    c.close()


def test_independent_groups_do_not_interfere():
    # two ring columns of a U2 x R2 mesh meet independently
    c = Comm.local(4)
    c.set_timeout(5)
    sig = "ring_shift(buffers=2,bytes=64,steps=1)"
    groups = {0: [0, 2], 2: [0, 2], 1: [1, 3], 3: [1, 3]}
    errs = _run_ranks([lambda r=r: [c.debug_rendezvous(r, groups[r], sig) for _ in range(4)] for r in range(4)])
    assert errs == [None] * 4
    c.close()


def test_timeout_validation():
    c = Comm.local(1)
    with pytest.raises(UspError):
        c.set_timeout(0)
    c.close()
