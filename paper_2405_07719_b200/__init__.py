"""B200-native Unified Sequence Parallelism (USP) attention forward and backward.

The product is libusp_b200.so (hand-written sm_100a CUDA + NCCL, C ABI in
include/usp_attn.h); this package is its host-side mirror of the reference
operator interface (see usp.py).
"""
from ._lib import UspError, UspInvalidInput, lib  # noqa: F401
from .usp import (  # noqa: F401
    Comm,
    ProcessMesh,
    ShardSpec,
    UspAttention,
    UspForward,
    UspGrads,
    causal_pair_counts,
    even_partition,
    local_world_backward,
    local_world_forward,
    usp_attention,
    zigzag_partition,
)

__version__ = "0.1.0"
