"""The reference's `uspsim_run` command interface (include/uspsim.h:33-55)
served by libusp_b200.so (include/usp_sim.h): a JSON request in, a report
(JSON document, text rendering, CSV communication ledger, exit code) out.

    >>> r = run({"command": "simulate", "params": {"seqlen": 4096, "heads": 8,
    ...          "head_size": 64, "ulysses": 2, "ring": 2, "causal": True,
    ...          "check": True}})
    >>> r.status, r.doc["results"]["check"]["passed"]

`simulate` runs every rank of the ulysses x ring mesh on the GPU (usp_attn_fwd
+ usp_attn_bwd over the in-process transport) and checks O, dQ, dK, dV
against an fp64 GPU reference, as src/api/commands.cpp:85-282 does on the CPU.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from typing import Optional, Union

from ._lib import lib

USPSIM_OK, USPSIM_TOLERANCE_EXCEEDED, USPSIM_INVALID_INPUT, USPSIM_INTERNAL_ERROR = 0, 1, 2, 3


@dataclass
class SimReport:
    status: int                 # uspsim_status returned by uspsim_run
    json: Optional[str]         # uspsim_report_json (None when no report was produced)
    text: str                   # uspsim_report_text, or uspsim_last_error() without a report
    ledger_csv: str
    exit_code: int

    @property
    def doc(self) -> dict:
        return json.loads(self.json) if self.json else {}


def run(request: Union[str, dict]) -> SimReport:
    """uspsim_run(request) -> report (freed before returning)."""
    req = request if isinstance(request, str) else json.dumps(request)
    L = lib()
    h = ctypes.c_void_p()
    st = int(L.uspsim_run(req.encode(), ctypes.byref(h)))
    if not h.value:
        return SimReport(st, None, L.uspsim_last_error().decode(), "", 2)
    try:
        return SimReport(st, L.uspsim_report_json(h).decode(), L.uspsim_report_text(h).decode(),
                         L.uspsim_report_ledger_csv(h).decode(), int(L.uspsim_report_exit_code(h)))
    finally:
        L.uspsim_report_free(h)
