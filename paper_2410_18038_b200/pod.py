"""Host-side mirror of the reference's hybrid-batch operator interface.

Same names and argument meaning as the reference's C++ API
(/root/reference/proj/include/attnsim/*.hpp), implemented over the C ABI of
libpod_attn.so.  Reference C++ exceptions become Python exceptions of the
same class names:

    std::invalid_argument -> InvalidArgument (ValueError)
    std::logic_error      -> LogicError
    std::domain_error     -> DomainError
    std::out_of_range     -> OutOfRange (IndexError)
    attnsim::ConfigError  -> ConfigError
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _abi
from ._abi import lib


class PodException(RuntimeError):
    status = -1


class InvalidArgument(PodException, ValueError):
    status = 1


class LogicError(PodException):
    status = 2


class DomainError(PodException, ValueError):
    status = 3


class OutOfRange(PodException, IndexError):
    status = 4


class ConfigError(PodException):
    status = 5


class CudaError(PodException):
    status = 6


class Unsupported(PodException, NotImplementedError):
    status = 7


_EXC = {c.status: c for c in (InvalidArgument, LogicError, DomainError, OutOfRange, ConfigError, CudaError,
                              Unsupported)}


def _check(status: int, where: str) -> None:
    if status != 0:
        msg = lib().pod_last_error().decode(errors="replace")
        raise _EXC.get(status, PodException)(f"{where}: {msg}")


# ----------------------------------------------------------------- types ---
@dataclass
class ModelShape:
    """ModelShape (types.hpp:60-76); `scale` is the softmax divisor."""
    num_q_heads: int = 32
    num_kv_heads: int = 4
    head_dim: int = 128
    scale: float = 11.313708498984761

    def group_size(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    def _c(self) -> _abi.pod_shape:
        return _abi.pod_shape(self.num_q_heads, self.num_kv_heads, self.head_dim, self.scale)


@dataclass
class PrefillSpec:
    """PrefillSpec (work_decomp.hpp:18-22)."""
    chunk_size: int = 0
    context_len: int = 0
    position_offset: int = 0


@dataclass
class DecodeSpec:
    """DecodeSpec (work_decomp.hpp:24-26)."""
    context_len: int = 0


@dataclass
class HybridBatchSpec:
    """HybridBatchSpec (work_decomp.hpp:28-48) + paged-KV layout of the GPU path."""
    prefill: Optional[PrefillSpec] = None
    decodes: List[DecodeSpec] = field(default_factory=list)
    shape: ModelShape = field(default_factory=ModelShape)
    page_size: int = 16
    kv_layout: int = _abi.POD_KV_HND
    dtype: int = _abi.POD_DTYPE_BF16

    def validate(self) -> None:
        """Raises InvalidArgument exactly where HybridBatchSpec::validate throws."""
        Plan(self, GpuSpec.reference_default()).close()

    def _c(self):
        ctx = (C.c_int64 * max(1, len(self.decodes)))(*[d.context_len for d in self.decodes])
        b = _abi.pod_batch()
        b.has_prefill = 1 if self.prefill is not None else 0
        if self.prefill is not None:
            b.prefill = _abi.pod_prefill_spec(self.prefill.chunk_size, self.prefill.context_len,
                                              self.prefill.position_offset)
        b.num_decodes = len(self.decodes)
        b.decode_context_len = C.cast(ctx, C.POINTER(C.c_int64))
        b.page_size = self.page_size
        b.kv_layout = self.kv_layout
        b.dtype = self.dtype
        return b, ctx


@dataclass
class GpuSpec:
    """GpuSpec (gpu.hpp:12-37)."""
    num_sms: int = 108
    compute_rate_per_sm: float = 0.25
    mem_bandwidth_total: float = 108.0
    mem_bandwidth_per_sm: float = 1.2
    mem_interference: float = 0.25
    max_ctas_per_sm: int = 4
    shared_mem_per_sm: float = 167936.0

    @staticmethod
    def reference_default() -> "GpuSpec":
        d = _abi.pod_device()
        lib().pod_device_reference_default(C.byref(d))
        return GpuSpec._from_c(d)

    @staticmethod
    def from_device(device: int = 0) -> "GpuSpec":
        d = _abi.pod_device()
        _check(lib().pod_device_query(device, C.byref(d)), "pod_device_query")
        return GpuSpec._from_c(d)

    @staticmethod
    def b200(num_sms: int = 148, head_dim: int = 128) -> "GpuSpec":
        """B200 calibration without a device."""
        tf, hbm = 1665.7e12, 6538.9e9
        tot = hbm / 2.0 / 1e6
        return GpuSpec(num_sms, tf / (4.0 * head_dim) / 1e6 / num_sms, tot, 1.2 * tot / num_sms, 0.25, 4,
                       232448.0)

    @staticmethod
    def _from_c(d) -> "GpuSpec":
        return GpuSpec(d.num_sms, d.compute_rate_per_sm, d.mem_bandwidth_total, d.mem_bandwidth_per_sm,
                       d.mem_interference, d.max_ctas_per_sm, d.shared_mem_per_sm)

    def _c(self) -> _abi.pod_device:
        return _abi.pod_device(self.num_sms, self.compute_rate_per_sm, self.mem_bandwidth_total,
                               self.mem_bandwidth_per_sm, self.mem_interference, self.max_ctas_per_sm,
                               self.shared_mem_per_sm)


@dataclass
class TileConfig:
    """TileConfig (work_decomp.hpp:50-60)."""
    prefill_tile_q: int = 128
    decode_tile_q: int = 16
    tile_kv: int = 64
    warps_per_cta: int = 4
    ctas_per_sm: int = 2
    shared_mem_per_cta: float = 65536.0
    virtual_decode: bool = False
    split_wave_cap: int = 2

    def _c(self) -> _abi.pod_tile_config:
        return _abi.pod_tile_config(self.prefill_tile_q, self.decode_tile_q, self.tile_kv, self.warps_per_cta,
                                    self.ctas_per_sm, self.shared_mem_per_cta, int(self.virtual_decode),
                                    self.split_wave_cap)

    @staticmethod
    def _from_c(c) -> "TileConfig":
        return TileConfig(c.prefill_tile_q, c.decode_tile_q, c.tile_kv, c.warps_per_cta, c.ctas_per_sm,
                          c.shared_mem_per_cta, bool(c.virtual_decode), c.split_wave_cap)


@dataclass
class CtaTask:
    """CtaTask (work_decomp.hpp:62-73); op 0 = prefill, 1 = decode."""
    op: int
    request_id: int
    kv_head: int
    q_tile: int
    kv_split: tuple
    is_virtual: bool
    compute_work: float
    memory_work: float
    barrier_segments: int
    slot_quanta: int


@dataclass
class WorkDecomposition:
    """WorkDecomposition (work_decomp.hpp:75-81)."""
    prefill_tasks: List[CtaTask]
    decode_tasks: List[CtaTask]
    config: TileConfig

    def total_tasks(self) -> int:
        return len(self.prefill_tasks) + len(self.decode_tasks)


@dataclass
class PlanOptions:
    policy: int = _abi.POD_POLICY_AUTO
    tile_mode: int = _abi.POD_TILE_B200
    ctas_per_sm: int = 0
    virtual_decode: int = -1
    split_wave_cap: int = 0
    decode_splits: int = 0
    tile_override: Optional[TileConfig] = None
    precision: int = _abi.POD_PRECISION_F16PV
    out_dtype: int = _abi.POD_OUT_F32
    prefill_tile_keys: int = 0  # warp-specialised pair engine: 0 = auto, 32 or 64
    prefill_s_buffers: int = 0  # 64-key pair engine: 0 = auto, 1 = single S (Q in TMEM), 2 = double S (Q in smem)


def _task(t) -> CtaTask:
    return CtaTask(t.op, t.request_id, t.kv_head, t.q_tile, (t.kv_begin, t.kv_end), bool(t.is_virtual),
                   t.compute_work, t.memory_work, t.barrier_segments, t.slot_quanta)


class Plan:
    """pod_attn_plan: host-only planning (decompose_hybrid + scheduler state)."""

    def __init__(self, batch: HybridBatchSpec, gpu: GpuSpec, options: Optional[PlanOptions] = None):
        options = options or PlanOptions()
        self.batch = batch
        self.gpu = gpu
        self.options = options
        cb, self._ctx_keep = batch._c()
        o = _abi.pod_options()
        lib().pod_options_default(C.byref(o))
        o.policy, o.tile_mode, o.ctas_per_sm = options.policy, options.tile_mode, options.ctas_per_sm
        o.virtual_decode, o.split_wave_cap, o.decode_splits = (options.virtual_decode, options.split_wave_cap,
                                                              options.decode_splits)
        o.precision = options.precision
        o.out_dtype = options.out_dtype
        o.prefill_tile_keys = options.prefill_tile_keys
        o.prefill_s_buffers = options.prefill_s_buffers
        tc = None
        if options.tile_override is not None:
            tc = options.tile_override._c()
            o.tile_override = C.pointer(tc)
        h = C.c_void_p()
        shape = batch.shape._c()
        dev = gpu._c()
        _check(lib().pod_attn_plan(C.byref(shape), C.byref(cb), C.byref(dev), C.byref(o), C.byref(h)),
               "pod_attn_plan")
        self.handle = h

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().pod_attn_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> _abi.pod_plan_info:
        i = _abi.pod_plan_info()
        _check(lib().pod_attn_plan_get_info(self.handle, C.byref(i)), "pod_attn_plan_get_info")
        return i

    def tile_config(self) -> TileConfig:
        return TileConfig._from_c(self.info().config)

    def tasks(self) -> WorkDecomposition:
        npf, nd = C.c_int64(0), C.c_int64(0)
        _check(lib().pod_attn_plan_tasks(self.handle, None, C.byref(npf), None, C.byref(nd)), "plan_tasks")
        pa = (_abi.pod_task * max(1, npf.value))()
        da = (_abi.pod_task * max(1, nd.value))()
        _check(lib().pod_attn_plan_tasks(self.handle, pa, C.byref(npf), da, C.byref(nd)), "plan_tasks")
        return WorkDecomposition([_task(pa[i]) for i in range(npf.value)],
                                 [_task(da[i]) for i in range(nd.value)], self.tile_config())

    def workspace_bytes(self) -> int:
        return int(lib().pod_attn_workspace_bytes(self.handle))


# ------------------------------------------- reference-named free functions --
def make_tile_config(ctas_per_sm: int) -> TileConfig:
    """make_tile_config (work_decomp.hpp:119-136)."""
    b = HybridBatchSpec(decodes=[DecodeSpec(1)], shape=ModelShape(1, 1, 128, 1.0))
    p = Plan(b, GpuSpec.reference_default(), PlanOptions(tile_mode=_abi.POD_TILE_REFERENCE,
                                                          ctas_per_sm=ctas_per_sm, virtual_decode=0))
    cfg = p.tile_config()
    p.close()
    return cfg


def select_tile_config(batch: HybridBatchSpec, gpu: GpuSpec) -> TileConfig:
    """select_tile_config (work_decomp.hpp:139-145)."""
    p = Plan(batch, gpu, PlanOptions(tile_mode=_abi.POD_TILE_REFERENCE, virtual_decode=-1))
    cfg = p.tile_config()
    p.close()
    return cfg


def decompose_hybrid(batch: HybridBatchSpec, gpu: GpuSpec, config: Optional[TileConfig] = None) -> WorkDecomposition:
    """decompose_hybrid (work_decomp.hpp:249-261)."""
    p = Plan(batch, gpu, PlanOptions(tile_mode=_abi.POD_TILE_REFERENCE, virtual_decode=-1, tile_override=config))
    wd = p.tasks()
    p.close()
    return wd


def limit_prefill_splits(natural_parallelism: int, gpu: GpuSpec, config: TileConfig) -> int:
    """limit_prefill_splits (work_decomp.hpp:147-155), through the planner: a prefill of
    `natural_parallelism` q tiles x 1 kv head reports its split count."""
    if natural_parallelism < 1:
        raise InvalidArgument("limit_prefill_splits: parallelism must be >= 1")
    cfg = TileConfig(**{**config.__dict__, "prefill_tile_q": 1, "tile_kv": 1})
    n = natural_parallelism
    b = HybridBatchSpec(prefill=PrefillSpec(n, n + 10 ** 6, 10 ** 6), shape=ModelShape(1, 1, 128, 1.0))
    p = Plan(b, gpu, PlanOptions(tile_mode=_abi.POD_TILE_REFERENCE, tile_override=cfg, virtual_decode=0))
    s = int(p.info().prefill_splits)
    p.close()
    return s


def gqa_kv_head(q_head: int, shape: ModelShape) -> int:
    """gqa_kv_head (attention.hpp:100-106)."""
    if q_head < 0 or q_head >= shape.num_q_heads:
        raise OutOfRange("gqa_kv_head: q_head out of range")
    return q_head // shape.group_size()


def split_ranges(n: int, splits: int):
    """split_ranges (attention.hpp:224-238)."""
    base, rem = divmod(n, splits)
    out, pos = [], 0
    for s in range(splits):
        ln = base + (1 if s < rem else 0)
        out.append((pos, pos + ln))
        pos += ln
    return out
