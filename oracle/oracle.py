"""ctypes front end for the parity checkers in oracle/.

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package
(paper_2405_07719_b200). Two libraries sit behind it:

* ``Oracle``    — liboracle_usp.so, the C restatement (usp_oracle.c) of the
  reference's forward; every entry cites the reference file:line it follows.
* ``Reference`` — _ref/libuspref.so, the reference's own sources compiled
  by oracle/Makefile (absent when /root/reference was not available at
  build time; callers must handle ``Reference.available() == False``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle_usp.so")
REF_SO = os.path.join(HERE, "_ref", "libuspref.so")
REF_SRC = "/root/reference/proj/src"

_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_int = ctypes.c_int


def build(ref: bool | None = None) -> None:
    """Compile liboracle_usp.so, and oracle/_ref when the reference exists."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _as(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


class _Lib:
    _lib = None
    path = ""

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(cls.path):
                build()
            cls._lib = ctypes.CDLL(cls.path)
            cls._declare(cls._lib)
        return cls._lib

    @classmethod
    def _declare(cls, lib):  # pragma: no cover - overridden
        raise NotImplementedError


class Oracle(_Lib):
    path = ORACLE_SO

    @classmethod
    def _declare(cls, lib):
        lib.uo_uniform_stream.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_double, _i64, _f64p]
        lib.uo_reference_attention.argtypes = [_f64p, _f64p, _f64p, _i64, _i64, _i64, _i64, _i64, _int,
                                               ctypes.c_void_p, _f64p]
        lib.uo_softmax_rows.argtypes = [_f64p, _f64p, _f64p, _i64, _i64, _i64, _i64, _i64, _i64, _int,
                                        _i64p, _i64p, _f64p, _f64p]
        lib.uo_softmax_rows.restype = _i64
        lib.uo_zigzag_partition.argtypes = [_i64, _int, _i64p]
        lib.uo_even_partition.argtypes = [_i64, _int, _i64p]
        lib.uo_causal_pair_counts.argtypes = [_i64p, _int, _i64, _i64p]
        lib.uo_positions_for.argtypes = [_int, _int, _i64, _int, _int, _i64p]
        lib.uo_usp_forward.argtypes = [_f64p, _f64p, _f64p, _i64, _i64, _i64, _i64, _i64, _int, _int, _int,
                                       _f64p, _f64p]

    # --- generators / layout -------------------------------------------------
    @classmethod
    def uniform(cls, seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        cls.lib().uo_uniform_stream(seed, lo, hi, n, out)
        return out

    @classmethod
    def zigzag_partition(cls, seq_len: int, ring: int) -> np.ndarray:
        out = np.empty(seq_len, np.int64)
        if cls.lib().uo_zigzag_partition(seq_len, ring, out) != 0:
            raise ValueError(f"sequence length {seq_len} is not divisible by 2*ring = {2 * ring}")
        return out.reshape(ring, seq_len // ring)

    @classmethod
    def even_partition(cls, seq_len: int, ring: int) -> np.ndarray:
        out = np.empty(seq_len, np.int64)
        if cls.lib().uo_even_partition(seq_len, ring, out) != 0:
            raise ValueError("sequence length is not divisible by the ring degree")
        return out.reshape(ring, seq_len // ring)

    @classmethod
    def causal_pair_counts(cls, assignment: np.ndarray, seq_len: int) -> np.ndarray:
        a = _as(assignment, np.int64)
        counts = np.empty(a.shape[0], np.int64)
        if cls.lib().uo_causal_pair_counts(a.reshape(-1), a.shape[0], seq_len, counts) != 0:
            raise ValueError("assignment must cover 0..L-1 exactly once")
        return counts

    @classmethod
    def positions_for(cls, ulysses: int, ring: int, seq_len: int, zigzag: bool, rank: int) -> np.ndarray:
        out = np.empty(seq_len // (ulysses * ring), np.int64)
        if cls.lib().uo_positions_for(ulysses, ring, seq_len, int(zigzag), rank, out) != 0:
            raise ValueError("invalid shard spec")
        return out

    # --- numerics -------------------------------------------------------------
    @classmethod
    def reference_attention(cls, q, k, v, causal: bool, positions=None) -> np.ndarray:
        q, k, v = _as(q), _as(k), _as(v)
        b, s, h, d = q.shape
        out = np.empty_like(q)
        pos = None
        if positions is not None:
            pos = _as(positions, np.int64)
        rc = cls.lib().uo_reference_attention(q, k, v, b, s, h, k.shape[2], d, int(causal),
                                              pos.ctypes.data if pos is not None else None, out)
        if rc != 0:
            raise ValueError("bad attention shapes")
        return out

    @classmethod
    def softmax_rows(cls, q, k, v, causal: bool, q_pos, k_pos):
        """O and natural-log LSE of query rows ``q`` (b, n, h, d) at original
        positions ``q_pos`` against keys at ``k_pos`` (one SoftmaxState update)."""
        q, k, v = _as(q), _as(k), _as(v)
        b, n, h, d = q.shape
        out = np.empty_like(q)
        lse = np.empty((b, n, h), np.float64)
        cls.lib().uo_softmax_rows(q, k, v, b, n, k.shape[1], h, k.shape[2], d, int(causal),
                                  _as(q_pos, np.int64), _as(k_pos, np.int64), out, lse)
        return out, lse

    @classmethod
    def usp_forward(cls, q, k, v, ulysses: int, ring: int, causal: bool):
        """Global O and per-rank head-sharded LSE blocks of usp_attention."""
        q, k, v = _as(q), _as(k), _as(v)
        b, s, h, d = q.shape
        kvh = k.shape[2]
        out = np.empty_like(q)
        n = ulysses * ring
        lse = np.empty((n, b, s // ring, h // ulysses), np.float64)
        if cls.lib().uo_usp_forward(q, k, v, b, s, h, kvh, d, ulysses, ring, int(causal), out, lse) != 0:
            raise ValueError("usp constraint violated")
        return out, lse


class Reference(_Lib):
    """The reference's own code (oracle/_ref/libuspref.so)."""

    path = REF_SO

    @classmethod
    def available(cls) -> bool:
        if os.path.exists(cls.path):
            return True
        if os.path.isdir(REF_SRC):
            try:
                build(ref=True)
            except Exception:
                return False
            return os.path.exists(cls.path)
        return False

    @classmethod
    def _declare(cls, lib):
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_last_ledger_json.restype = ctypes.c_char_p
        lib.ref_uniform_stream.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_double, _i64, _f64p]
        lib.ref_reference_attention_f64.argtypes = [_f64p, _f64p, _f64p, _i64, _i64, _i64, _i64, _i64, _int,
                                                    ctypes.c_void_p, _f64p]
        for name in ("ref_softmax_rows_f64", "ref_softmax_rows_f32"):
            getattr(lib, name).argtypes = [_f64p, _f64p, _f64p, _i64, _i64, _i64, _i64, _i64, _i64, _int,
                                           _i64p, _i64p, _f64p, _f64p]
        lib.ref_zigzag_partition.argtypes = [_i64, _int, _i64p]
        lib.ref_positions_for.argtypes = [_int, _int, _i64, _int, _int, _i64p]
        lib.ref_causal_pair_counts.argtypes = [_i64p, _int, _i64, _i64p]
        for name in ("ref_usp_forward_f64", "ref_usp_forward_f32"):
            getattr(lib, name).argtypes = [_f64p, _f64p, _f64p, _i64, _i64, _i64, _i64, _i64, _int, _int, _int,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]

    @classmethod
    def _check(cls, rc):
        if rc != 0:
            msg = cls.lib().ref_last_error().decode()
            raise ValueError(msg)

    @classmethod
    def uniform(cls, seed: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        cls.lib().ref_uniform_stream(seed, lo, hi, n, out)
        return out

    @classmethod
    def reference_attention(cls, q, k, v, causal: bool, positions=None) -> np.ndarray:
        q, k, v = _as(q), _as(k), _as(v)
        b, s, h, d = q.shape
        out = np.empty_like(q)
        pos = _as(positions, np.int64) if positions is not None else None
        cls._check(cls.lib().ref_reference_attention_f64(q, k, v, b, s, h, k.shape[2], d, int(causal),
                                                         pos.ctypes.data if pos is not None else None, out))
        return out

    @classmethod
    def softmax_rows(cls, q, k, v, causal: bool, q_pos, k_pos, precision: str = "fp64"):
        """The reference's SoftmaxState<T>::update + finalize + logsumexp of
        query rows ``q`` against keys ``k_pos``; precision "fp32" runs
        SoftmaxState<float> on the float-cast inputs (the reference's fp32
        path), results widened to fp64."""
        q, k, v = _as(q), _as(k), _as(v)
        b, n, h, d = q.shape
        out = np.empty_like(q)
        lse = np.empty((b, n, h), np.float64)
        fn = cls.lib().ref_softmax_rows_f64 if precision == "fp64" else cls.lib().ref_softmax_rows_f32
        cls._check(fn(q, k, v, b, n, k.shape[1], h, k.shape[2], d, int(causal),
                                                  _as(q_pos, np.int64), _as(k_pos, np.int64), out, lse))
        return out, lse

    @classmethod
    def zigzag_partition(cls, seq_len: int, ring: int) -> np.ndarray:
        out = np.empty(seq_len, np.int64)
        cls._check(cls.lib().ref_zigzag_partition(seq_len, ring, out))
        return out.reshape(ring, seq_len // ring)

    @classmethod
    def positions_for(cls, ulysses: int, ring: int, seq_len: int, zigzag: bool, rank: int) -> np.ndarray:
        out = np.empty(seq_len // (ulysses * ring), np.int64)
        cls._check(cls.lib().ref_positions_for(ulysses, ring, seq_len, int(zigzag), rank, out))
        return out

    @classmethod
    def causal_pair_counts(cls, assignment: np.ndarray, seq_len: int) -> np.ndarray:
        a = _as(assignment, np.int64)
        counts = np.empty(a.shape[0], np.int64)
        cls._check(cls.lib().ref_causal_pair_counts(a.reshape(-1), a.shape[0], seq_len, counts))
        return counts

    @classmethod
    def usp_forward(cls, q, k, v, ulysses: int, ring: int, causal: bool, precision: str = "fp64",
                    want_out: bool = True):
        """Runs the reference usp_attention<T> on U*R rank threads. Returns
        (out_global, lse_blocks, seconds_in_World_run)."""
        q, k, v = _as(q), _as(k), _as(v)
        b, s, h, d = q.shape
        out = np.empty_like(q) if want_out else None
        lse = np.empty((ulysses * ring, b, s // ring, h // ulysses), np.float64) if want_out else None
        secs = ctypes.c_double(0.0)
        fn = cls.lib().ref_usp_forward_f64 if precision == "fp64" else cls.lib().ref_usp_forward_f32
        cls._check(fn(q, k, v, b, s, h, k.shape[2], d, ulysses, ring, int(causal),
                      out.ctypes.data if out is not None else None,
                      lse.ctypes.data if lse is not None else None, ctypes.byref(secs)))
        return out, lse, secs.value

    @classmethod
    def last_ledger(cls):
        """The reference World's CommLedger entries of the last usp_forward."""
        import json

        return json.loads(cls.lib().ref_last_ledger_json().decode())


# ---- backward -------------------------------------------

def _declare_bwd(lib, prefix):
    fp, ip = _f64p, ctypes.c_void_p
    if prefix == "uo":
        lib.uo_reference_attention_grad.argtypes = [fp, fp, fp, fp, _i64, _i64, _i64, _i64, _i64, _int, ip,
                                                    fp, fp, fp]
        lib.uo_usp_backward.argtypes = [fp, fp, fp, fp, _i64, _i64, _i64, _i64, _i64, _int, _int, _int,
                                        fp, fp, fp]
    else:
        lib.ref_reference_attention_grad_f64.argtypes = [fp, fp, fp, fp, _i64, _i64, _i64, _i64, _i64, _int, ip,
                                                         fp, fp, fp]
        lib.ref_usp_fwd_bwd_f64.argtypes = [fp, fp, fp, fp, _i64, _i64, _i64, _i64, _i64, _int, _int, _int,
                                            fp, fp, fp]


def _grad_call(fn, q, k, v, dout, causal, positions=None, mesh=None):
    q, k, v, dout = _as(q), _as(k), _as(v), _as(dout)
    b, s, h, d = q.shape
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    if mesh is None:
        pos = _as(positions, np.int64) if positions is not None else None
        rc = fn(q, k, v, dout, b, s, h, k.shape[2], d, int(causal), pos.ctypes.data if pos is not None else None,
                dq, dk, dv)
    else:
        rc = fn(q, k, v, dout, b, s, h, k.shape[2], d, mesh[0], mesh[1], int(causal), dq, dk, dv)
    return rc, (dq, dk, dv)


def oracle_reference_attention_grad(q, k, v, dout, causal, positions=None):
    lib = Oracle.lib()
    _declare_bwd(lib, "uo")
    rc, g = _grad_call(lib.uo_reference_attention_grad, q, k, v, dout, causal, positions)
    if rc != 0:
        raise ValueError("bad attention shapes")
    return g


def oracle_usp_backward(q, k, v, dout, ulysses, ring, causal):
    lib = Oracle.lib()
    _declare_bwd(lib, "uo")
    rc, g = _grad_call(lib.uo_usp_backward, q, k, v, dout, causal, mesh=(ulysses, ring))
    if rc != 0:
        raise ValueError("usp constraint violated")
    return g


def reference_attention_grad(q, k, v, dout, causal, positions=None):
    lib = Reference.lib()
    _declare_bwd(lib, "ref")
    rc, g = _grad_call(lib.ref_reference_attention_grad_f64, q, k, v, dout, causal, positions)
    Reference._check(rc)
    return g


def reference_usp_fwd_bwd(q, k, v, dout, ulysses, ring, causal):
    lib = Reference.lib()
    _declare_bwd(lib, "ref")
    rc, g = _grad_call(lib.ref_usp_fwd_bwd_f64, q, k, v, dout, causal, mesh=(ulysses, ring))
    Reference._check(rc)
    return g
