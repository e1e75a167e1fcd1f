"""paper_2410_18038_b200 -- B200-native POD-Attention (arXiv 2410.18038) hot path.

One sm_100a launch computes the prefill-chunk attention and the paged decode
attention of a hybrid batch concurrently (SM-aware CTA role binding), behind
the C ABI in include/pod_attn.h.  This package holds the kernels (csrc/), the
in-tree build, and a host mirror of the reference's operator interface.
"""
from ._abi import LIB_PATH, lib  # noqa: F401
from .pod import (  # noqa: F401
    ConfigError, CtaTask, DecodeSpec, DomainError, GpuSpec, HybridBatchSpec, InvalidArgument, LogicError,
    ModelShape, OutOfRange, Plan, PlanOptions, PrefillSpec, TileConfig, Unsupported, WorkDecomposition,
    decompose_hybrid, gqa_kv_head, limit_prefill_splits, make_tile_config, select_tile_config, split_ranges,
)

__all__ = [
    "ModelShape", "PrefillSpec", "DecodeSpec", "HybridBatchSpec", "GpuSpec", "TileConfig", "CtaTask",
    "WorkDecomposition", "Plan", "PlanOptions", "decompose_hybrid", "select_tile_config", "make_tile_config",
    "limit_prefill_splits", "gqa_kv_head", "split_ranges", "PodAttention",
]


def __getattr__(name):
    if name == "PodAttention":
        from .hybrid import PodAttention
        return PodAttention
    raise AttributeError(name)
