"""Host-side mirror of the reference's USP operator interface.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/src), so code written against it reads the same:

  ProcessMesh            src/simcomm/mesh.hpp:14-34
  zigzag_partition,
  even_partition,
  causal_pair_counts,
  ShardSpec              src/usp/partition.hpp:19-53
  usp_attention          src/usp/usp_attention.hpp:41-47  (forward)
  UspForward             src/usp/usp_attention.hpp:16-24  (out + logsumexp + head_positions)

Constraint violations raise ``UspInvalidInput`` (a ValueError) carrying the
reference's message ("... cannot exceed ...", "... not divisible by 2*ring
..."). All compute goes through the C ABI of libusp_b200.so (hand-written
sm_100a kernels); torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from ._lib import UspConfig, UspError, UspInvalidInput, UspLedgerEntry, UspStepInfo, check, lib

__all__ = [
    "ProcessMesh", "ShardSpec", "zigzag_partition", "even_partition", "causal_pair_counts",
    "Comm", "UspAttention", "UspForward", "usp_attention", "UspError", "UspInvalidInput",
    "make_config",
]


# ------------------------------------------------------------------ layout
class ProcessMesh:
    """rank = ring_coord * U + ulysses_coord; rows are Ulysses groups,
    columns are Ring groups (mesh.hpp:9-13)."""

    def __init__(self, ulysses_degree: int, ring_degree: int):
        if ulysses_degree < 1 or ring_degree < 1:
            raise UspInvalidInput(2, "mesh degrees must be >= 1")
        self.ulysses = int(ulysses_degree)
        self.ring = int(ring_degree)

    def ulysses_degree(self) -> int:
        return self.ulysses

    def ring_degree(self) -> int:
        return self.ring

    def world_size(self) -> int:
        return self.ulysses * self.ring

    def _check(self, rank: int) -> None:
        if rank < 0 or rank >= self.world_size():
            raise UspInvalidInput(2, f"rank {rank} outside mesh of size {self.world_size()}")

    def ulysses_coord(self, rank: int) -> int:
        self._check(rank)
        return rank % self.ulysses

    def ring_coord(self, rank: int) -> int:
        self._check(rank)
        return rank // self.ulysses

    def rank_of(self, ulysses_coord: int, ring_coord: int) -> int:
        if not (0 <= ulysses_coord < self.ulysses and 0 <= ring_coord < self.ring):
            raise UspInvalidInput(2, "mesh coordinates out of range")
        return ring_coord * self.ulysses + ulysses_coord

    def ulysses_group(self, rank: int) -> list[int]:
        r = self.ring_coord(rank)
        return [self.rank_of(u, r) for u in range(self.ulysses)]

    def ring_group(self, rank: int) -> list[int]:
        u = self.ulysses_coord(rank)
        return [self.rank_of(u, r) for r in range(self.ring)]


def zigzag_partition(seq_len: int, ring_degree: int) -> list[list[int]]:
    out = np.empty(seq_len, np.int64)
    check(lib().usp_zigzag_partition(seq_len, ring_degree, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return out.reshape(ring_degree, -1).tolist()


def even_partition(seq_len: int, ring_degree: int) -> list[list[int]]:
    if ring_degree < 1:
        raise UspInvalidInput(2, "ring degree must be >= 1")
    if seq_len % ring_degree:
        raise UspInvalidInput(2, "sequence length is not divisible by the ring degree")
    return np.arange(seq_len, dtype=np.int64).reshape(ring_degree, -1).tolist()


def causal_pair_counts(assignment: Sequence[Sequence[int]], seq_len: int) -> list[int]:
    flat = np.ascontiguousarray(np.asarray(assignment, dtype=np.int64).reshape(-1))
    ring = len(assignment)
    if flat.size != seq_len:
        raise UspInvalidInput(2, "assignment must cover 0..L-1 exactly once")
    counts = np.empty(ring, np.int64)
    p = ctypes.POINTER(ctypes.c_int64)
    check(lib().usp_causal_pair_counts(flat.ctypes.data_as(p), ring, seq_len, counts.ctypes.data_as(p)))
    return counts.tolist()


def make_config(mesh: ProcessMesh, *, rank: int, seq_len: int, heads: int, kv_heads: int,
                head_size: int, causal: bool, batch: int = 1, device: int = 0) -> UspConfig:
    return UspConfig(mesh.ulysses, mesh.ring, rank, device, batch, seq_len, heads, kv_heads,
                     head_size, int(bool(causal)))


class ShardSpec:
    """Each ring rank's token list (zigzag iff ``zigzag``) cut into U
    sub-shards, one per Ulysses rank (partition.hpp:32-53)."""

    def __init__(self, mesh: ProcessMesh, seq_len: int, zigzag: bool):
        self.mesh = mesh
        self.seq_len = int(seq_len)
        self.zigzag = bool(zigzag)
        # Shape checks only (heads are validated by the engine).
        cfg = make_config(mesh, rank=0, seq_len=seq_len, heads=mesh.ulysses, kv_heads=mesh.ulysses,
                          head_size=64, causal=zigzag)
        check(lib().usp_config_validate(ctypes.byref(cfg)))
        self._cfg = cfg

    def tokens_per_rank(self) -> int:
        return self.seq_len // self.mesh.world_size()

    def positions_for(self, rank: int) -> list[int]:
        out = np.empty(self.tokens_per_rank(), np.int64)
        check(lib().usp_positions_for(ctypes.byref(self._cfg), rank,
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out.tolist()

    def head_positions(self, rank: int) -> list[int]:
        out = np.empty(self.seq_len // self.mesh.ring, np.int64)
        check(lib().usp_head_positions(ctypes.byref(self._cfg), rank,
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out.tolist()


def schedule(cfg: UspConfig, step: int) -> UspStepInfo:
    info = UspStepInfo()
    check(lib().usp_schedule(ctypes.byref(cfg), step, ctypes.byref(info)))
    return info


def step_plan(cfg: UspConfig, step: int):
    """(tile_off, tile_list) CSR of one ring step's tile plan."""
    sizes = (ctypes.c_int64 * 2)()
    check(lib().usp_step_plan(ctypes.byref(cfg), step, sizes, None, None))
    off = np.empty(sizes[0] + 1, np.int32)
    lst = np.empty(max(sizes[1], 1), np.int32)
    p32 = ctypes.POINTER(ctypes.c_int32)
    check(lib().usp_step_plan(ctypes.byref(cfg), step, sizes, off.ctypes.data_as(p32), lst.ctypes.data_as(p32)))
    return off, lst[: sizes[1]]


def _read_ledger(call) -> list[dict]:
    """Two-pass read of a ledger C function (cap 0 returns the size)."""
    n = call(None, 0)
    if n < 0:
        check(2)
    buf = (UspLedgerEntry * max(n, 1))()
    m = call(buf, n)
    if m < 0:
        check(2)
    return [buf[i].as_dict() for i in range(min(m, n))]


def forward_ledger(cfg: UspConfig) -> list[dict]:
    """Planned collectives of one rank's forward (reference CommLedger terms)."""
    return _read_ledger(lambda buf, cap: lib().usp_forward_ledger(ctypes.byref(cfg), buf, cap))


def backward_ledger(cfg: UspConfig) -> list[dict]:
    """Planned collectives of one rank's forward + backward
    (usp_attention.cpp:68-89, ring_attention.cpp:79-155)."""
    return _read_ledger(lambda buf, cap: lib().usp_backward_ledger(ctypes.byref(cfg), buf, cap))


def rank_flops(cfg: UspConfig) -> float:
    f = ctypes.c_double(0)
    check(lib().usp_rank_flops(ctypes.byref(cfg), ctypes.byref(f)))
    return f.value


# --------------------------------------------------------------- transports
class Comm:
    """A transport between the ranks of one mesh (usp_comm)."""

    def __init__(self, handle: int, kind: str, world_size: int):
        self._h = ctypes.c_void_p(handle)
        self.kind = kind
        self.world_size = world_size

    @classmethod
    def local(cls, world_size: int) -> "Comm":
        """In-process world: one host thread per rank (simcomm::World analogue)."""
        h = ctypes.c_void_p()
        check(lib().usp_comm_create_local(world_size, ctypes.byref(h)))
        return cls(h.value, "local", world_size)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib().usp_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, unique_id: bytes, world_size: int, rank: int, device: int) -> "Comm":
        h = ctypes.c_void_p()
        check(lib().usp_comm_create_nccl(unique_id, world_size, rank, device, ctypes.byref(h)))
        return cls(h.value, "nccl", world_size)

    @classmethod
    def from_torch_distributed(cls, device: int, group=None) -> "Comm":
        """NCCL transport over the ranks of a torch.distributed group: rank 0
        draws the ncclUniqueId and broadcasts it (torch is plumbing here)."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = cls.nccl_unique_id() if rank == 0 else bytes(128)
        backend = dist.get_backend(group)
        dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=0, group=group)
        return cls.nccl(bytes(t.cpu().tolist()), world, rank, device)

    @classmethod
    def p2p(cls, world_size: int, rank: int, device: int, allgather) -> "Comm":
        """Peer-memory transport (usp_comm_create_p2p): CUDA IPC buffers written
        directly by the senders with copy engines, no NCCL. ``allgather(bytes)
        -> list[bytes]`` is a host all-gather over the world in rank order; it
        is called collectively at creation and when a buffer is first used."""
        from ._lib import ALLGATHER_FN

        def _cb(send, recv, nbytes, _ctx):
            try:
                parts = allgather(ctypes.string_at(send, nbytes))
                if len(parts) != world_size or any(len(x) != nbytes for x in parts):
                    return 1
                ctypes.memmove(recv, b"".join(parts), nbytes * world_size)
                return 0
            except Exception:  # pragma: no cover - reported as a failed collective
                return 1

        cb = ALLGATHER_FN(_cb)
        h = ctypes.c_void_p()
        check(lib().usp_comm_create_p2p(world_size, rank, device, cb, None, ctypes.byref(h)))
        c = cls(h.value, "p2p", world_size)
        c._keep = cb  # the library calls it for the comm's whole lifetime
        return c

    @classmethod
    def p2p_from_torch_distributed(cls, device: int, group=None) -> "Comm":
        """The peer-memory transport bootstrapped over a torch.distributed
        group (a gloo group is created for the host all-gather when the
        given one is not CPU-capable)."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        host_group = group if dist.get_backend(group) == "gloo" else dist.new_group(backend="gloo")

        def allgather(blob: bytes):
            t = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t, group=host_group)
            return [bytes(x.numpy().tobytes()) for x in out]

        return cls.p2p(world, rank, device, allgather)

    def set_timeout(self, seconds: float) -> None:
        """How long a collective may wait for its peers before the comm
        reports it (usp_comm_set_timeout)."""
        check(lib().usp_comm_set_timeout(self._h, float(seconds)))

    def status(self) -> None:
        """Raises UspError with the failure if the comm has failed."""
        check(lib().usp_comm_status(self._h))

    def debug_rendezvous(self, rank: int, members: Sequence[int], signature: str) -> None:
        """Tests: one host rendezvous (local transport) without GPU work."""
        arr = (ctypes.c_int32 * len(members))(*members)
        check(lib().usp_comm_debug_rendezvous(self._h, rank, arr, len(members), signature.encode()))

    def close(self) -> None:
        if self._h:
            lib().usp_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------- engine
@dataclass
class UspForward:
    """Forward results (usp_attention.hpp:16-24): ``out`` sequence-sharded
    like the inputs; ``logsumexp`` head-sharded (batch, L/R, heads/U),
    natural log, rows in ``head_positions`` order."""

    out: "object"
    logsumexp: "object"
    head_positions: list
    # the forward's inputs (the engine keeps their head-sharded copies)
    q: "object" = None
    k: "object" = None
    v: "object" = None


@dataclass
class UspGrads:
    """Backward results (usp_attention.hpp:26-31): dq, dk, dv sequence-sharded
    like q, k, v (bf16)."""

    dq: "object"
    dk: "object"
    dv: "object"


def _ptr(t) -> int:
    return int(t.data_ptr())


class UspAttention:
    """One rank's USP forward engine (usp_engine): workspace, comms and the
    per-step tile plans are built once; ``forward`` is collective over the
    mesh and asynchronous on the given CUDA stream."""

    def __init__(self, mesh: ProcessMesh, *, rank: int, seq_len: int, heads: int, kv_heads: int,
                 head_size: int, causal: bool, batch: int = 1, device: int = 0,
                 comm: Optional[Comm] = None):
        self.mesh = mesh
        self.rank = rank
        self.cfg = make_config(mesh, rank=rank, seq_len=seq_len, heads=heads, kv_heads=kv_heads,
                               head_size=head_size, causal=causal, batch=batch, device=device)
        check(lib().usp_config_validate(ctypes.byref(self.cfg)))
        self.comm = comm
        h = ctypes.c_void_p()
        check(lib().usp_engine_create(ctypes.byref(self.cfg), comm._h if comm else None, ctypes.byref(h)))
        self._h = h
        self.batch, self.seq_len, self.heads, self.kv_heads = batch, seq_len, heads, kv_heads
        self.head_size, self.causal, self.device = head_size, bool(causal), device
        self.tokens = seq_len // mesh.world_size()

    # shapes
    def q_shape(self):
        return (self.batch, self.tokens, self.heads, self.head_size)

    def kv_shape(self):
        return (self.batch, self.tokens, self.kv_heads, self.head_size)

    def lse_shape(self):
        return (self.batch, self.seq_len // self.mesh.ring, self.heads // self.mesh.ulysses)

    def head_positions(self) -> list[int]:
        out = np.empty(self.seq_len // self.mesh.ring, np.int64)
        check(lib().usp_head_positions(ctypes.byref(self.cfg), self.rank,
                                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out.tolist()

    def positions(self) -> list[int]:
        out = np.empty(self.tokens, np.int64)
        check(lib().usp_positions_for(ctypes.byref(self.cfg), self.rank,
                                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out.tolist()

    def flops(self) -> float:
        return rank_flops(self.cfg)

    def last_launches(self) -> int:
        return int(lib().usp_engine_last_launches(self._h))

    def ledger(self) -> list[dict]:
        """Collectives issued by the last forward (reference CommLedger terms)."""
        return _read_ledger(lambda buf, cap: lib().usp_engine_ledger(self._h, buf, cap))

    def info(self) -> dict:
        """Ring overlap sizing (usp_engine_get_info)."""
        from ._lib import UspEngineInfo

        i = UspEngineInfo()
        check(lib().usp_engine_get_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in i._fields_}

    def set_a2a_chunks(self, chunks: int) -> None:
        """Row chunks of the pipelined Ulysses all-to-alls (1 = one exchange
        each way; default 2 where it applies, see usp_engine_set_a2a_chunks)."""
        check(lib().usp_engine_set_a2a_chunks(self._h, int(chunks)))

    @property
    def a2a_chunks(self) -> int:
        return int(lib().usp_engine_a2a_chunks(self._h))

    def set_deterministic(self, on: bool = True) -> None:
        """Backward algorithm: fused one-kernel (default; dQ reduced in fp32
        in arrival order, last bits may vary run to run) or the
        bitwise-reproducible two-kernel path (``on=True``)."""
        check(lib().usp_engine_set_deterministic(self._h, 1 if on else 0))

    def set_reserved_sms(self, n: int) -> None:
        check(lib().usp_engine_set_reserved_sms(self._h, int(n)))

    def stage_times(self) -> list[dict]:
        """Per-stage breakdown of the forwards timed since enable_timing:
        [{"stage", "ms_total", "count"}] (usp_engine_stage_times); syncs."""
        from ._lib import UspStageTime

        cap = 512
        buf = (UspStageTime * cap)()
        n = int(lib().usp_engine_stage_times(self._h, buf, cap))
        if n < 0:
            check(3)
        return [{"stage": buf[i].name.decode(), "ms_total": buf[i].ms_total, "count": buf[i].count}
                for i in range(min(n, cap))]

    def debug_counters(self, on: bool = True) -> None:
        """Parity instrumentation: count the forward kernel's lazy O rescales
        (resets the count)."""
        check(lib().usp_engine_debug_counters(self._h, int(on)))

    def rescale_count(self) -> int:
        """(warp, key tile) rescales of O since debug_counters(True); syncs."""
        out = ctypes.c_int64()
        check(lib().usp_engine_rescale_count(self._h, ctypes.byref(out)))
        return int(out.value)

    def enable_timing(self, on: bool = True) -> None:
        """Record CUDA events around every attention-kernel launch."""
        check(lib().usp_engine_enable_timing(self._h, int(on)))

    def kernel_times(self) -> list[float]:
        """Durations (ms) of the attention launches since the last call."""
        cap = 1 << 16
        buf = (ctypes.c_float * cap)()
        n = int(lib().usp_engine_kernel_times(self._h, buf, cap))
        if n < 0:
            check(3)
        return list(buf[:min(n, cap)])

    def _check_tensors(self, q, k, v, out, lse):
        import torch

        for name, t, shape, dt in (("q", q, self.q_shape(), torch.bfloat16),
                                   ("k", k, self.kv_shape(), torch.bfloat16),
                                   ("v", v, self.kv_shape(), torch.bfloat16),
                                   ("out", out, self.q_shape(), torch.bfloat16),
                                   ("lse", lse, self.lse_shape(), torch.float32)):
            if tuple(t.shape) != tuple(shape) or t.dtype != dt or not t.is_cuda or not t.is_contiguous():
                raise UspInvalidInput(2, f"{name} must be a contiguous {dt} CUDA tensor of shape {shape}, "
                                         f"got {tuple(t.shape)} {t.dtype} on {t.device}")

    def alloc_outputs(self):
        import torch

        dev = torch.device("cuda", self.device)
        return (torch.empty(self.q_shape(), dtype=torch.bfloat16, device=dev),
                torch.empty(self.lse_shape(), dtype=torch.float32, device=dev))

    def forward(self, q, k, v, out=None, lse=None, stream=None) -> UspForward:
        import torch

        if out is None or lse is None:
            o2, l2 = self.alloc_outputs()
            out = o2 if out is None else out
            lse = l2 if lse is None else lse
        self._check_tensors(q, k, v, out, lse)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().usp_attn_fwd(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse),
                                 ctypes.c_void_p(s.cuda_stream)))
        return UspForward(out, lse, self.head_positions(), q, k, v)

    __call__ = forward

    def forward_host(self, q, k, v, out, lse, stream=None) -> UspForward:
        """usp_attn_fwd_host: the forward with q, k, v, out, lse in host
        memory (pinned CPU tensors for copy/compute overlap); the host<->device
        copies run inside the call, pipelined against the attention in
        sequence chunks at U = R = 1. ``out``/``lse`` are valid after the
        stream is synchronised."""
        import torch

        for name, t, shape, dt in (("q", q, self.q_shape(), torch.bfloat16),
                                   ("k", k, self.kv_shape(), torch.bfloat16),
                                   ("v", v, self.kv_shape(), torch.bfloat16),
                                   ("out", out, self.q_shape(), torch.bfloat16),
                                   ("lse", lse, self.lse_shape(), torch.float32)):
            if tuple(t.shape) != tuple(shape) or t.dtype != dt or t.is_cuda or not t.is_contiguous():
                raise UspInvalidInput(2, f"{name} must be a contiguous {dt} host tensor of shape {shape}, "
                                         f"got {tuple(t.shape)} {t.dtype} on {t.device}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().usp_attn_fwd_host(self._h, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse),
                                      ctypes.c_void_p(s.cuda_stream)))
        return UspForward(out, lse, self.head_positions(), None, None, None)

    def alloc_grads(self):
        import torch

        dev = torch.device("cuda", self.device)
        return (torch.empty(self.q_shape(), dtype=torch.bfloat16, device=dev),
                torch.empty(self.kv_shape(), dtype=torch.bfloat16, device=dev),
                torch.empty(self.kv_shape(), dtype=torch.bfloat16, device=dev))

    def _check_bwd(self, fwd: UspForward, dout, dq, dk, dv):
        import torch

        if fwd.q is None:
            raise UspInvalidInput(2, "logsumexp does not match the forward shard (missing forward artifacts?)")
        self._check_tensors(fwd.q, fwd.k, fwd.v, fwd.out, fwd.logsumexp)
        for name, t, shape in (("dout", dout, self.q_shape()), ("dq", dq, self.q_shape()),
                               ("dk", dk, self.kv_shape()), ("dv", dv, self.kv_shape())):
            if tuple(t.shape) != tuple(shape) or t.dtype != torch.bfloat16 or not t.is_cuda \
                    or not t.is_contiguous():
                what = "dO must be sequence-sharded like the forward output" if name == "dout" else \
                    f"{name} must be a contiguous bfloat16 CUDA tensor of shape {shape}"
                raise UspInvalidInput(2, f"{what}, got {tuple(t.shape)} {t.dtype} on {t.device}")

    def backward(self, fwd: UspForward, dout, dq=None, dk=None, dv=None, stream=None) -> UspGrads:
        """usp_attention_backward (usp_attention.cpp:68-89) of the engine's
        most recent forward ``fwd``; collective over the mesh."""
        import torch

        if dq is None or dk is None or dv is None:
            a, b, c = self.alloc_grads()
            dq, dk, dv = (dq if dq is not None else a), (dk if dk is not None else b), (dv if dv is not None else c)
        self._check_bwd(fwd, dout, dq, dk, dv)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().usp_attn_bwd(self._h, _ptr(fwd.q), _ptr(fwd.k), _ptr(fwd.v), _ptr(fwd.out),
                                 _ptr(fwd.logsumexp), _ptr(dout), _ptr(dq), _ptr(dk), _ptr(dv),
                                 ctypes.c_void_p(s.cuda_stream)))
        return UspGrads(dq, dk, dv)

    def close(self) -> None:
        if self._h:
            lib().usp_engine_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def local_world_forward(engines: Sequence[UspAttention], qs, ks, vs, outs, lses, streams) -> None:
    """usp_attn_fwd on every rank of an in-process world (one host thread
    per rank inside the library), like simcomm::World::run."""
    n = len(engines)
    arr = lambda xs: (ctypes.c_void_p * n)(*[ctypes.c_void_p(x) for x in xs])  # noqa: E731
    check(lib().usp_local_world_fwd(arr([e._h.value for e in engines]), n, arr(map(_ptr, qs)),
                                    arr(map(_ptr, ks)), arr(map(_ptr, vs)), arr(map(_ptr, outs)),
                                    arr(map(_ptr, lses)), arr([s.cuda_stream for s in streams])))


def local_world_backward(engines: Sequence[UspAttention], fwds: Sequence[UspForward], douts, dqs, dks, dvs,
                         streams) -> None:
    """usp_attn_bwd on every rank of an in-process world."""
    n = len(engines)
    arr = lambda xs: (ctypes.c_void_p * n)(*[ctypes.c_void_p(x) for x in xs])  # noqa: E731
    check(lib().usp_local_world_bwd(arr([e._h.value for e in engines]), n, arr(_ptr(f.q) for f in fwds),
                                    arr(_ptr(f.k) for f in fwds), arr(_ptr(f.v) for f in fwds),
                                    arr(_ptr(f.out) for f in fwds), arr(_ptr(f.logsumexp) for f in fwds),
                                    arr(map(_ptr, douts)), arr(map(_ptr, dqs)), arr(map(_ptr, dks)),
                                    arr(map(_ptr, dvs)), arr([s.cuda_stream for s in streams])))


# usp_attention() reuses one engine per configuration (workspace, plans and
# the transport's sub-communicators are built once, as a layer would).
_ENGINE_CACHE: "dict[tuple, UspAttention]" = {}
_ENGINE_CACHE_SIZE = 8


def usp_attention(mesh: ProcessMesh, q, k, v, positions: Sequence[int], causal: bool, *,
                  rank: int, seq_len: int, comm: Optional[Comm] = None, device: int = 0) -> UspForward:
    """Functional form of the reference's usp_attention (usp_attention.hpp:41-47)
    for one rank. ``positions`` must be ShardSpec(mesh, L, causal).positions_for(rank),
    the only layout the reference produces; the engine checks it."""
    b, t, hc, hs = q.shape
    key = (mesh.ulysses, mesh.ring, rank, seq_len, hc, k.shape[2], hs, bool(causal), b, device, id(comm))
    eng = _ENGINE_CACHE.pop(key, None)
    if eng is None:
        eng = UspAttention(mesh, rank=rank, seq_len=seq_len, heads=hc, kv_heads=k.shape[2], head_size=hs,
                           causal=causal, batch=b, device=device, comm=comm)
    _ENGINE_CACHE[key] = eng  # most recently used last
    while len(_ENGINE_CACHE) > _ENGINE_CACHE_SIZE:
        _ENGINE_CACHE.pop(next(iter(_ENGINE_CACHE))).close()
    if list(positions) != eng.positions():
        raise UspInvalidInput(2, "positions must carry one original index per local token "
                                 "in ShardSpec::positions_for order")
    return eng.forward(q, k, v)
