"""ctypes binding of libusp_b200.so (the C ABI in include/usp_attn.h).

There is no fallback: if the native library is missing and cannot be built
(no nvcc), importing the engine raises. The library is built in-tree by
build.py so it travels with the repository snapshot.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("USPB_LIB_PATH") or os.path.join(HERE, "libusp_b200.so")  # override: dev A/B builds

USP_OK, USP_TOLERANCE_EXCEEDED, USP_INVALID_INPUT, USP_INTERNAL_ERROR = 0, 1, 2, 3


class UspError(RuntimeError):
    """A non-OK usp_status; ``status`` mirrors uspsim_status numbering."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class UspInvalidInput(UspError, ValueError):
    pass


class UspConfig(ctypes.Structure):
    _fields_ = [
        ("ulysses_degree", ctypes.c_int32),
        ("ring_degree", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("batch", ctypes.c_int64),
        ("seq_len", ctypes.c_int64),
        ("heads", ctypes.c_int32),
        ("kv_heads", ctypes.c_int32),
        ("head_size", ctypes.c_int32),
        ("causal", ctypes.c_int32),
    ]


class UspStepInfo(ctypes.Structure):
    _fields_ = [
        ("step", ctypes.c_int32),
        ("src_ring_coord", ctypes.c_int32),
        ("send_to_rank", ctypes.c_int32),
        ("recv_from_rank", ctypes.c_int32),
        ("full_tiles", ctypes.c_int64),
        ("partial_tiles", ctypes.c_int64),
        ("work_units", ctypes.c_int64),
        ("visible_pairs", ctypes.c_int64),
        ("ring_bytes_sent", ctypes.c_int64),
    ]


class UspLedgerEntry(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("group_first", ctypes.c_int32),
        ("group_size", ctypes.c_int32),
        ("group_stride", ctypes.c_int32),
        ("step", ctypes.c_int32),
        ("tensor", ctypes.c_int32),
        ("payload_elems", ctypes.c_int64),
        ("bytes_sent", ctypes.c_double),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class UspEngineInfo(ctypes.Structure):
    _fields_ = [("num_sms", ctypes.c_int32), ("reserved_sms", ctypes.c_int32), ("ring_ctas", ctypes.c_int32),
                ("kv_shift_bytes", ctypes.c_double), ("ring_step_ms_est", ctypes.c_double),
                ("required_gbs", ctypes.c_double)]


class UspStageTime(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("ms_total", ctypes.c_double), ("count", ctypes.c_int32)]


# Every symbol include/usp_attn.h declares (tests check the .so exports them).
EXPORTS = [
    "usp_config_validate", "usp_zigzag_partition", "usp_positions_for", "usp_head_positions",
    "usp_causal_pair_counts", "usp_schedule", "usp_step_plan", "usp_forward_ledger", "usp_engine_ledger", "usp_rank_flops", "usp_nccl_unique_id",
    "usp_comm_create_nccl", "usp_comm_create_local", "usp_comm_destroy", "usp_engine_create",
    "usp_attn_fwd", "usp_engine_last_launches", "usp_engine_destroy", "usp_engine_enable_timing",
    "usp_engine_kernel_times", "usp_engine_debug_counters", "usp_engine_rescale_count",
    "usp_engine_stage_times", "usp_engine_get_info", "usp_engine_set_reserved_sms", "usp_engine_set_deterministic", "usp_engine_set_a2a_chunks", "usp_engine_a2a_chunks", "usp_comm_set_timeout", "usp_comm_status", "usp_comm_debug_rendezvous", "usp_local_world_fwd", "usp_attn_bwd", "usp_local_world_bwd",
    "usp_backward_ledger", "usp_attn_fwd_host", "usp_comm_create_p2p",
    "usp_last_error", "usp_version",
]
# Every symbol include/usp_sim.h declares (the reference's uspsim.h ABI).
SIM_EXPORTS = [
    "uspsim_run", "uspsim_report_json", "uspsim_report_text", "uspsim_report_ledger_csv",
    "uspsim_report_exit_code", "uspsim_report_free", "uspsim_last_error", "uspsim_version",
]

# int (*)(const void* send, void* recv, size_t bytes, void* ctx)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)

_lib = None
_lock = threading.Lock()


def _declare(lib):
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    st = ctypes.c_int
    i64p = P(ctypes.c_int64)
    sig = {
        "usp_config_validate": (st, [P(UspConfig)]),
        "usp_zigzag_partition": (st, [ctypes.c_int64, ctypes.c_int32, i64p]),
        "usp_positions_for": (st, [P(UspConfig), ctypes.c_int32, i64p]),
        "usp_head_positions": (st, [P(UspConfig), ctypes.c_int32, i64p]),
        "usp_causal_pair_counts": (st, [i64p, ctypes.c_int32, ctypes.c_int64, i64p]),
        "usp_schedule": (st, [P(UspConfig), ctypes.c_int32, P(UspStepInfo)]),
        "usp_step_plan": (st, [P(UspConfig), ctypes.c_int32, i64p, P(ctypes.c_int32), P(ctypes.c_int32)]),
        "usp_rank_flops": (st, [P(UspConfig), P(ctypes.c_double)]),
        "usp_forward_ledger": (ctypes.c_int32, [P(UspConfig), P(UspLedgerEntry), ctypes.c_int32]),
        "usp_engine_ledger": (ctypes.c_int32, [vp, P(UspLedgerEntry), ctypes.c_int32]),
        "usp_backward_ledger": (ctypes.c_int32, [P(UspConfig), P(UspLedgerEntry), ctypes.c_int32]),
        "usp_attn_bwd": (st, [vp] * 11),
        "usp_local_world_bwd": (st, [P(vp), ctypes.c_int32] + [P(vp)] * 10),
        "usp_nccl_unique_id": (st, [ctypes.c_char_p]),
        "usp_comm_create_nccl": (st, [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P(vp)]),
        "usp_comm_create_local": (st, [ctypes.c_int32, P(vp)]),
        "usp_comm_create_p2p": (st, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ALLGATHER_FN, vp, P(vp)]),
        "usp_comm_destroy": (None, [vp]),
        "usp_comm_set_timeout": (st, [vp, ctypes.c_double]),
        "usp_comm_status": (st, [vp]),
        "usp_comm_debug_rendezvous": (st, [vp, ctypes.c_int32, P(ctypes.c_int32), ctypes.c_int32, ctypes.c_char_p]),
        "usp_engine_create": (st, [P(UspConfig), vp, P(vp)]),
        "usp_attn_fwd": (st, [vp, vp, vp, vp, vp, vp, vp]),
        "usp_attn_fwd_host": (st, [vp, vp, vp, vp, vp, vp, vp]),
        "usp_engine_last_launches": (ctypes.c_int32, [vp]),
        "usp_engine_destroy": (None, [vp]),
        "usp_engine_enable_timing": (st, [vp, ctypes.c_int32]),
        "usp_engine_kernel_times": (ctypes.c_int32, [vp, P(ctypes.c_float), ctypes.c_int32]),
        "usp_engine_debug_counters": (st, [vp, ctypes.c_int32]),
        "usp_engine_stage_times": (ctypes.c_int32, [vp, P(UspStageTime), ctypes.c_int32]),
        "usp_engine_get_info": (st, [vp, P(UspEngineInfo)]),
        "usp_engine_set_reserved_sms": (st, [vp, ctypes.c_int32]),
        "usp_engine_set_deterministic": (st, [vp, ctypes.c_int32]),
        "usp_engine_set_a2a_chunks": (st, [vp, ctypes.c_int32]),
        "usp_engine_a2a_chunks": (ctypes.c_int32, [vp]),
        "usp_engine_rescale_count": (st, [vp, i64p]),
        "usp_local_world_fwd": (st, [P(vp), ctypes.c_int32, P(vp), P(vp), P(vp), P(vp), P(vp), P(vp)]),
        "usp_last_error": (ctypes.c_char_p, []),
        "uspsim_run": (st, [ctypes.c_char_p, P(vp)]),
        "uspsim_report_json": (ctypes.c_char_p, [vp]),
        "uspsim_report_text": (ctypes.c_char_p, [vp]),
        "uspsim_report_ledger_csv": (ctypes.c_char_p, [vp]),
        "uspsim_report_exit_code": (ctypes.c_int, [vp]),
        "uspsim_report_free": (None, [vp]),
        "uspsim_last_error": (ctypes.c_char_p, []),
        "uspsim_version": (ctypes.c_char_p, []),
        "usp_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """Loads (building first if needed) libusp_b200.so."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                from . import build as _build  # nvcc is required: no CPU fallback

                _build.build()
            _lib = ctypes.CDLL(LIB_PATH)
            _declare(_lib)
    return _lib


def check(status: int) -> None:
    if status == USP_OK:
        return
    msg = lib().usp_last_error().decode()
    if status == USP_INVALID_INPUT:
        raise UspInvalidInput(status, msg)
    raise UspError(status, msg)
