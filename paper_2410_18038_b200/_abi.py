"""ctypes view of the C ABI in include/pod_attn.h.

The product path is libpod_attn.so (sm_100a kernels + host planner).  Loading
fails loudly if the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libpod_attn.so"

POD_OK = 0
STATUS_NAMES = {
    0: "ok", 1: "invalid_argument", 2: "logic_error", 3: "domain_error",
    4: "out_of_range", 5: "config_error", 6: "cuda_error", 7: "unsupported",
}

POD_KV_HND, POD_KV_NHD = 0, 1
POD_DTYPE_BF16, POD_DTYPE_FP16 = 0, 1
POD_POLICY_FIFTY_FIFTY, POD_POLICY_PROPORTIONAL, POD_POLICY_CLAMPED, POD_POLICY_COMPLEMENT = 0, 1, 2, 3
# 4-6 retired (measured slower; pod_attn_plan rejects them)
POD_POLICY_WARPSPEC, POD_POLICY_AUTO = 7, 8
POD_TILE_REFERENCE, POD_TILE_B200 = 0, 1
POD_PRECISION_SPLIT, POD_PRECISION_FAST, POD_PRECISION_F16PV = 0, 1, 2
POD_OUT_F32, POD_OUT_BF16, POD_OUT_F16 = 0, 1, 2


class pod_shape(C.Structure):
    _fields_ = [("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("scale", C.c_double)]


class pod_prefill_spec(C.Structure):
    _fields_ = [("chunk_size", C.c_int64), ("context_len", C.c_int64),
                ("position_offset", C.c_int64)]


class pod_batch(C.Structure):
    _fields_ = [("has_prefill", C.c_int32), ("prefill", pod_prefill_spec),
                ("num_decodes", C.c_int64), ("decode_context_len", C.POINTER(C.c_int64)),
                ("page_size", C.c_int32), ("kv_layout", C.c_int32), ("dtype", C.c_int32)]


class pod_device(C.Structure):
    _fields_ = [("num_sms", C.c_int32), ("compute_rate_per_sm", C.c_double),
                ("mem_bandwidth_total", C.c_double), ("mem_bandwidth_per_sm", C.c_double),
                ("mem_interference", C.c_double), ("max_ctas_per_sm", C.c_int32),
                ("shared_mem_per_sm", C.c_double)]


class pod_tile_config(C.Structure):
    _fields_ = [("prefill_tile_q", C.c_int64), ("decode_tile_q", C.c_int64),
                ("tile_kv", C.c_int64), ("warps_per_cta", C.c_int32),
                ("ctas_per_sm", C.c_int32), ("shared_mem_per_cta", C.c_double),
                ("virtual_decode", C.c_int32), ("split_wave_cap", C.c_int32)]


class pod_task(C.Structure):
    _fields_ = [("op", C.c_int32), ("request_id", C.c_int32), ("kv_head", C.c_int32),
                ("q_tile", C.c_int32), ("kv_begin", C.c_int64), ("kv_end", C.c_int64),
                ("is_virtual", C.c_int32), ("slot_quanta", C.c_int32),
                ("barrier_segments", C.c_int64), ("compute_work", C.c_double),
                ("memory_work", C.c_double)]


class pod_options(C.Structure):
    _fields_ = [("policy", C.c_int32), ("tile_mode", C.c_int32), ("ctas_per_sm", C.c_int32),
                ("virtual_decode", C.c_int32), ("split_wave_cap", C.c_int32),
                ("decode_splits", C.c_int32), ("tile_override", C.POINTER(pod_tile_config)),
                ("precision", C.c_int32), ("out_dtype", C.c_int32), ("prefill_tile_keys", C.c_int32),
                ("prefill_s_buffers", C.c_int32)]


class pod_plan_info(C.Structure):
    _fields_ = [("config", pod_tile_config), ("prefill_splits", C.c_int64),
                ("num_prefill_tasks", C.c_int64), ("num_decode_tasks", C.c_int64),
                ("num_prefill_ctas", C.c_int64), ("num_decode_ctas", C.c_int64),
                ("decode_splits", C.c_int64), ("prefill_ratio", C.c_int64),
                ("decode_ratio", C.c_int64), ("smem_bytes", C.c_int64),
                ("workspace_bytes", C.c_int64), ("num_merge_rows_prefill", C.c_int32),
                ("num_merge_rows_decode", C.c_int32), ("policy", C.c_int32), ("prefill_tile_keys", C.c_int32),
                ("prefill_s_buffers", C.c_int32)]


# (name, restype, argtypes) for every symbol include/pod_attn.h declares.
_vp = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_fp = C.POINTER(C.c_float)
SYMBOLS = [
    ("pod_device_query", C.c_int, [C.c_int, C.POINTER(pod_device)]),
    ("pod_device_reference_default", None, [C.POINTER(pod_device)]),
    ("pod_options_default", None, [C.POINTER(pod_options)]),
    ("pod_attn_plan", C.c_int, [C.POINTER(pod_shape), C.POINTER(pod_batch), C.POINTER(pod_device),
                                C.POINTER(pod_options), C.POINTER(_vp)]),
    ("pod_attn_plan_destroy", None, [_vp]),
    ("pod_attn_plan_get_info", C.c_int, [_vp, C.POINTER(pod_plan_info)]),
    ("pod_attn_plan_tasks", C.c_int, [_vp, C.POINTER(pod_task), C.POINTER(C.c_int64),
                                      C.POINTER(pod_task), C.POINTER(C.c_int64)]),
    ("pod_attn_workspace_bytes", C.c_size_t, [_vp]),
    ("pod_attn_workspace_init", C.c_int, [_vp, _vp, _vp]),
    ("pod_attn_run", C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("pod_attn_run_serial", C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("pod_attn_run_part", C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp]),
    ("pod_attn_set_role_log", C.c_int, [_vp, _vp]),
    ("pod_attn_l2_flush", C.c_int, [_vp, C.c_int64, _vp]),
    ("pod_oproj_run", C.c_int, [_vp, _vp, C.c_int64, C.c_int64, C.c_int64, C.POINTER(_vp), C.c_int32, C.c_int64,
                                C.c_int32, _vp]),
    ("pod_attn_gather_probe", C.c_int, [_vp, _vp, C.c_int64, _vp, _vp, C.c_int32, C.c_int64, _vp, _vp]),
    ("pod_attn_append_kv", C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int64, _vp, _vp, _vp, _vp]),
    ("pod_attn_occupancy", C.c_int, [_vp, _i32p, _i32p, _i32p]),
    ("pod_status_string", C.c_char_p, [C.c_int]),
    ("pod_last_error", C.c_char_p, []),
    ("pod_attn_abi_version", C.c_int, []),
]

_lib = None


def lib() -> C.CDLL:
    """Loads libpod_attn.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        path = Path(os.environ["POD_LIB"]) if os.environ.get("POD_LIB") else LIB_PATH  # experiment builds
        if not path.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the POD kernels)")
        l = C.CDLL(str(path))
        for name, res, args in SYMBOLS:
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


class PodError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().pod_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)} ({msg})")
        self.status = status


def check(status: int, where: str) -> None:
    if status != POD_OK:
        raise PodError(status, where)
