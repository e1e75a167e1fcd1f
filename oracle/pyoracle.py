"""TEST INFRASTRUCTURE ONLY: ctypes bindings to the two CPU checkers.

  port() -> oracle/liboracle.so          plain-C restatement (pod_oracle.c)
  ref()  -> oracle/_ref/libattnsim_ref.so the reference's own headers compiled
                                          in place (ref_shim.cpp, oracle/Makefile)

All arrays are numpy float64 / int64 (contiguous).  Status codes follow
include/pod_attn.h (1 invalid_argument, 2 logic_error, 3 domain_error,
4 out_of_range).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_PATH = HERE / "liboracle.so"
REF_PATH = HERE / "_ref" / "libattnsim_ref.so"

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_long)
_i64p = C.POINTER(C.c_int64)

_port = None
_ref = None


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: status {status}")
        self.status = status


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def port() -> C.CDLL:
    global _port
    if _port is None:
        if not PORT_PATH.exists():
            raise ImportError(f"{PORT_PATH} missing: run `make -C oracle`")
        l = C.CDLL(str(PORT_PATH))
        l.orc_tiled_prefill.argtypes = [_dp, C.c_long, C.c_long, _dp, _dp, C.c_long, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_long, C.c_long, _dp]
        l.orc_prefill_lse.argtypes = [_dp, C.c_long, C.c_long, _dp, C.c_long, C.c_int, C.c_int, C.c_int,
                                      C.c_double, _dp]
        l.orc_decode_splitk.argtypes = [_dp, _dp, _dp, C.c_long, C.c_int, C.c_int, C.c_int, C.c_double, C.c_long,
                                        _dp, _dp, _lp, _lp]
        l.orc_merge_partials.argtypes = [_dp, _dp, _lp, C.c_long, C.c_long, C.c_long, _dp, _dp]
        l.orc_decode_attention.argtypes = [_dp, _dp, _dp, C.c_long, C.c_int, C.c_int, C.c_int, C.c_double, _dp,
                                           _dp]
        l.orc_naive_attention.argtypes = [_dp, C.c_long, _dp, _dp, C.c_long, C.c_long, C.c_double, C.c_int,
                                          C.c_long, _dp]
        l.orc_split_ranges.argtypes = [C.c_long, C.c_long, _lp, _lp]
        l.orc_gqa_kv_head.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        l.orc_gather_pages.argtypes = [C.c_void_p, C.c_int, C.c_long, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                       C.c_void_p, C.c_int, C.c_long, _dp]
        l.orc_append_kv.argtypes = [C.c_void_p, C.c_int, C.c_long, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_int, C.c_long, C.c_long, C.c_void_p]
        l.orc_append_kv.restype = C.c_int
        l.orc_sched_ratio.argtypes = [C.c_int, C.c_long, C.c_long, _lp, _lp]
        l.orc_sm_aware_replay.argtypes = [C.c_long, C.c_long, C.c_long, C.c_long, C.c_int, C.c_void_p, C.c_long,
                                          C.c_void_p, C.c_void_p]
        for f in ("orc_tiled_prefill", "orc_prefill_lse", "orc_decode_splitk", "orc_merge_partials",
                  "orc_decode_attention", "orc_naive_attention", "orc_gqa_kv_head", "orc_gather_pages"):
            getattr(l, f).restype = C.c_int
        _port = l
    return _port


def ref_available() -> bool:
    return REF_PATH.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            raise ImportError(f"{REF_PATH} missing: run `make -C oracle` where /root/reference exists")
        l = C.CDLL(str(REF_PATH))
        l.ref_rng_doubles.argtypes = [C.c_uint64, C.c_int64, _dp]
        l.ref_rng_longs.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, _i64p]
        l.ref_tiled_prefill.argtypes = [_dp, C.c_int64, C.c_int64, _dp, _dp, C.c_int64, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_int64, C.c_int64, _dp]
        l.ref_decode_splitk.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_int64, _dp, _dp, _i64p, _i64p]
        l.ref_merge_partials.argtypes = [_dp, _dp, _i64p, C.c_int64, C.c_int64, C.c_int64, _dp]
        l.ref_naive_attention.argtypes = [_dp, C.c_int64, _dp, _dp, C.c_int64, C.c_int64, C.c_double, C.c_int,
                                          C.c_int64, _dp]
        l.ref_decode_attention.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double, _dp]
        l.ref_split_ranges.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        l.ref_gqa_kv_head.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        l.ref_run_shards.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_int64, C.c_int64, C.c_int,
                                     C.POINTER(C.c_int)]
        l.ref_run_shards.restype = C.c_double
        l.ref_sched_replay.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_int64, _i64p, _i64p,
                                       C.c_void_p, C.c_void_p]
        l.ref_generate_trace.argtypes = [C.c_double, C.c_int64, C.c_int, C.c_double, C.c_double, C.c_int,
                                         C.c_double, C.c_double, C.c_uint64, _dp, _i64p, _i64p]
        l.ref_run_serving_linear.argtypes = [C.c_int64, _dp, _i64p, _i64p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                             C.c_double, C.c_double, C.c_int64, _dp, _dp, _i64p, _i64p, _i64p,
                                             _i64p, _dp, _dp, _dp]
        l.ref_generate_trace.restype = C.c_int
        l.ref_run_serving_linear.restype = C.c_int
        for f in ("ref_tiled_prefill", "ref_decode_splitk", "ref_merge_partials", "ref_naive_attention",
                  "ref_decode_attention", "ref_gqa_kv_head", "ref_decompose_hybrid", "ref_select_tile_config",
                  "ref_limit_prefill_splits", "ref_make_tile_config"):
            getattr(l, f).restype = C.c_int
        _ref = l
    return _ref


def _lib(which: str):
    return port() if which == "port" else ref()


# ------------------------------------------------------------- attention ---
def tiled_prefill(q, k, v, offset, hq, hkv, scale, tile_q, tile_kv, which="port"):
    """q [chunk][hq][d], k/v [ctx][hkv][d] -> O [chunk][hq][d]."""
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    chunk, _, d = q.shape
    out = np.zeros((chunk, hq, d), np.float64)
    fn = port().orc_tiled_prefill if which == "port" else ref().ref_tiled_prefill
    st = fn(_d(q), chunk, offset, _d(k), _d(v), k.shape[0], hq, hkv, d, scale, tile_q, tile_kv, _d(out))
    if st:
        raise OracleError(st, "tiled_prefill")
    return out


def prefill_lse(q, k, offset, hq, hkv, scale):
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    chunk, _, d = q.shape
    out = np.zeros((chunk, hq), np.float64)
    st = port().orc_prefill_lse(_d(q), chunk, offset, _d(k), k.shape[0], hq, hkv, d, scale, _d(out))
    if st:
        raise OracleError(st, "prefill_lse")
    return out


def decode_splitk(q, k, v, hq, hkv, scale, num_splits, which="port"):
    """q [hq][d] -> (o_parts [n][hq][d], lse_parts [n][hq], ranges [n][2])."""
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    d = q.shape[-1]
    ctx = k.shape[0]
    n = max(1, min(num_splits, max(ctx, 1)))
    o = np.zeros((n, hq, d), np.float64)
    lse = np.zeros((n, hq), np.float64)
    if which == "port":
        rg = np.zeros((n, 2), np.int64)
        cnt = C.c_long(0)
        st = port().orc_decode_splitk(_d(q), _d(k), _d(v), ctx, hq, hkv, d, scale, num_splits, _d(o), _d(lse),
                                      rg.ctypes.data_as(_lp), C.byref(cnt))
    else:
        rg = np.zeros((n, 2), np.int64)
        cnt = C.c_int64(0)
        st = ref().ref_decode_splitk(_d(q), _d(k), _d(v), ctx, hq, hkv, d, scale, num_splits, _d(o), _d(lse),
                                     rg.ctypes.data_as(_i64p), C.byref(cnt))
    if st:
        raise OracleError(st, "decode_splitk")
    c = cnt.value
    return o[:c], lse[:c], rg[:c]


def merge_partials(o_parts, lse_parts, ranges, which="port", with_lse=False):
    o_parts = np.ascontiguousarray(o_parts, np.float64)
    lse_parts = np.ascontiguousarray(lse_parts, np.float64)
    ranges = np.ascontiguousarray(ranges, np.int64)
    n = o_parts.shape[0] if o_parts.ndim == 3 else 0
    rows, d = (o_parts.shape[1], o_parts.shape[2]) if n else (0, 0)
    out = np.zeros((rows, d), np.float64)
    lse = np.zeros(rows, np.float64)
    if which == "port":
        st = port().orc_merge_partials(_d(o_parts), _d(lse_parts), ranges.ctypes.data_as(_lp), n, rows, d, _d(out),
                                       _d(lse))
    else:
        st = ref().ref_merge_partials(_d(o_parts), _d(lse_parts), ranges.ctypes.data_as(_i64p), n, rows, d,
                                      _d(out))
    if st:
        raise OracleError(st, "merge_partials")
    return (out, lse) if with_lse else out


def decode_attention(q, k, v, hq, hkv, scale, which="port"):
    """-> (O [hq][d], lse [hq]) for one decode request (LSE only from the port)."""
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    d = q.shape[-1]
    out = np.zeros((hq, d), np.float64)
    lse = np.zeros(hq, np.float64)
    if which == "port":
        st = port().orc_decode_attention(_d(q), _d(k), _d(v), k.shape[0], hq, hkv, d, scale, _d(out), _d(lse))
    else:
        st = ref().ref_decode_attention(_d(q), _d(k), _d(v), k.shape[0], hq, hkv, d, scale, _d(out))
        lse = None
    if st:
        raise OracleError(st, "decode_attention")
    return out, lse


def naive_attention(q, k, v, scale, causal_offset=None, which="port"):
    q = np.ascontiguousarray(q, np.float64)
    k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    m, d = q.shape
    out = np.zeros((m, d), np.float64)
    has = 0 if causal_offset is None else 1
    off = 0 if causal_offset is None else causal_offset
    fn = port().orc_naive_attention if which == "port" else ref().ref_naive_attention
    st = fn(_d(q), m, _d(k), _d(v), k.shape[0], d, scale, has, off, _d(out))
    if st:
        raise OracleError(st, "naive_attention")
    return out


def split_ranges(n, splits, which="port"):
    b = np.zeros(splits, np.int64)
    e = np.zeros(splits, np.int64)
    if which == "port":
        port().orc_split_ranges(n, splits, b.ctypes.data_as(_lp), e.ctypes.data_as(_lp))
    else:
        ref().ref_split_ranges(n, splits, b.ctypes.data_as(_i64p), e.ctypes.data_as(_i64p))
    return list(zip(b.tolist(), e.tolist()))


def gqa_kv_head(q_head, hq, hkv, which="port"):
    out = C.c_int(0)
    fn = port().orc_gqa_kv_head if which == "port" else ref().ref_gqa_kv_head
    st = fn(q_head, hq, hkv, C.byref(out))
    if st:
        raise OracleError(st, "gqa_kv_head")
    return out.value


def gather_pages(pool_u16: np.ndarray, layout: int, page_indptr: np.ndarray, page_indices: np.ndarray,
                 req: int, ctx: int) -> np.ndarray:
    """pool [num_pages][...] uint16 bf16 bits -> contiguous [ctx][hkv][d] float64."""
    pool_u16 = np.ascontiguousarray(pool_u16, np.uint16)
    if layout == 0:
        num_pages, hkv, ps, d = pool_u16.shape
    else:
        num_pages, ps, hkv, d = pool_u16.shape
    ip = np.ascontiguousarray(page_indptr, np.int32)
    ix = np.ascontiguousarray(page_indices, np.int32)
    out = np.zeros((ctx, hkv, d), np.float64)
    st = port().orc_gather_pages(pool_u16.ctypes.data, layout, num_pages, hkv, ps, d, ip.ctypes.data,
                                 ix.ctypes.data, req, ctx, _d(out))
    if st:
        raise OracleError(st, "gather_pages")
    return out


def append_kv(pool_u16: np.ndarray, layout: int, page_indptr: np.ndarray, page_indices: np.ndarray,
              req: int, pos0: int, rows_u16: np.ndarray) -> None:
    """In place: rows [ntok][hkv][d] (16-bit words) -> positions pos0.. of request req."""
    assert pool_u16.flags.c_contiguous and pool_u16.dtype == np.uint16
    if layout == 0:
        num_pages, hkv, ps, d = pool_u16.shape
    else:
        num_pages, ps, hkv, d = pool_u16.shape
    rows = np.ascontiguousarray(rows_u16, np.uint16)
    ip = np.ascontiguousarray(page_indptr, np.int32)
    ix = np.ascontiguousarray(page_indices, np.int32)
    st = port().orc_append_kv(pool_u16.ctypes.data, layout, num_pages, hkv, ps, d, ip.ctypes.data, ix.ctypes.data,
                              req, pos0, rows.shape[0], rows.ctypes.data)
    if st:
        raise OracleError(st, "append_kv")


def sched_replay(proportional: int, p_total: int, d_total: int, num_sms: int, sm_ids, which="port"):
    sm = np.ascontiguousarray(sm_ids, np.int32)
    n = len(sm)
    ops = np.zeros(n, np.int32)
    ids = np.zeros(n, np.int64)
    if which == "port":
        pr, dr = C.c_long(0), C.c_long(0)
        port().orc_sched_ratio(proportional, p_total, d_total, C.byref(pr), C.byref(dr))
        port().orc_sm_aware_replay(pr.value, dr.value, p_total, d_total, num_sms, sm.ctypes.data, n,
                                   ops.ctypes.data, ids.ctypes.data)
    else:
        pr, dr = C.c_int64(0), C.c_int64(0)
        ref().ref_sched_replay(proportional, p_total, d_total, num_sms, sm.ctypes.data, n, C.byref(pr),
                               C.byref(dr), ops.ctypes.data, ids.ctypes.data)
    return (pr.value, dr.value), ops, ids


def rng_doubles(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float64)
    ref().ref_rng_doubles(seed, n, _d(out))
    return out


# ---------------------------------------------------------- planner (ref) ---
class RefTask(C.Structure):
    _fields_ = [("op", C.c_int32), ("request_id", C.c_int32), ("kv_head", C.c_int32), ("q_tile", C.c_int32),
                ("kv_begin", C.c_int64), ("kv_end", C.c_int64), ("is_virtual", C.c_int32),
                ("slot_quanta", C.c_int32), ("barrier_segments", C.c_int64), ("compute_work", C.c_double),
                ("memory_work", C.c_double)]


class RefTileConfig(C.Structure):
    _fields_ = [("prefill_tile_q", C.c_int64), ("decode_tile_q", C.c_int64), ("tile_kv", C.c_int64),
                ("warps_per_cta", C.c_int32), ("ctas_per_sm", C.c_int32), ("shared_mem_per_cta", C.c_double),
                ("virtual_decode", C.c_int32), ("split_wave_cap", C.c_int32)]


class RefGpuSpec(C.Structure):
    _fields_ = [("num_sms", C.c_int32), ("compute_rate_per_sm", C.c_double), ("mem_bandwidth_total", C.c_double),
                ("mem_bandwidth_per_sm", C.c_double), ("mem_interference", C.c_double),
                ("max_ctas_per_sm", C.c_int32), ("shared_mem_per_sm", C.c_double)]


def ref_decompose_hybrid(shape, prefill, decode_ctx, gpu, cfg=None):
    """shape (hq, hkv, d, scale); prefill (chunk, prompt, offset) or None; gpu RefGpuSpec;
    cfg RefTileConfig or None (select_tile_config).  -> (status, cfg, prefill_tasks, decode_tasks)."""
    hq, hkv, d, scale = shape
    nd = len(decode_ctx)
    ctx = (C.c_int64 * max(1, nd))(*decode_ctx)
    cap_p = 1 << 16
    cap_d = max(16, nd * hkv * 64)
    pt = (RefTask * cap_p)()
    dt = (RefTask * cap_d)()
    np_, nd_ = C.c_int64(cap_p), C.c_int64(cap_d)
    out_cfg = RefTileConfig()
    has = 1 if prefill is not None else 0
    ch, pr, off = prefill if prefill is not None else (0, 0, 0)
    l = ref()
    st = l.ref_decompose_hybrid(hq, hkv, d, C.c_double(scale), has, C.c_int64(ch), C.c_int64(pr), C.c_int64(off),
                                C.c_int64(nd), ctx, C.byref(gpu), C.byref(cfg) if cfg is not None else None,
                                C.byref(out_cfg), pt, C.byref(np_), dt, C.byref(nd_))
    return st, out_cfg, [pt[i] for i in range(np_.value)] if not st else [], \
        [dt[i] for i in range(nd_.value)] if not st else []


DES_FIELDS = ("serial", "fused_best", "oracle_runtime", "prefill_alone", "decode_alone", "ctas_per_sm",
              "streams", "fused_selected")


def ref_des_predict(shape, prefill, decode_ctx, gpu):
    """The reference's discrete-event model of one hybrid batch (gpu_sim.hpp:781-816):
    dict of DES_FIELDS (times in the GpuSpec's time unit)."""
    hq, hkv, d, scale = shape
    nd = len(decode_ctx)
    ctx = (C.c_int64 * max(1, nd))(*decode_ctx)
    has = 1 if prefill is not None else 0
    ch, pr, off = prefill if prefill is not None else (0, 0, 0)
    out = (C.c_double * 8)()
    st = ref().ref_des_predict(hq, hkv, d, C.c_double(scale), has, C.c_int64(ch), C.c_int64(pr),
                               C.c_int64(off), C.c_int64(nd), ctx, C.byref(gpu), out)
    if st:
        raise OracleError(f"ref_des_predict: status {st}")
    return dict(zip(DES_FIELDS, list(out)))


def ref_limit_prefill_splits(natural, gpu, cfg):
    out = C.c_int64(0)
    st = ref().ref_limit_prefill_splits(C.c_int64(natural), C.byref(gpu), C.byref(cfg), C.byref(out))
    return st, out.value


# ------------------------------------------------------ CPU baseline shards --
class RefShard(C.Structure):
    _fields_ = [("kind", C.c_int32), ("group", C.c_int32), ("rows", C.c_int64), ("offset", C.c_int64),
                ("ctx", C.c_int64), ("q", _dp), ("k", _dp), ("v", _dp), ("out", _dp)]


def run_shards(shards, d, scale, tile_q, tile_kv, threads):
    """shards: list of dicts with kind, group, rows, offset, q, k, v, out (numpy float64).
    Runs the reference's tiled_prefill_attention / decode_attention over them with the
    reference's parallel_for; returns seconds."""
    arr = (RefShard * len(shards))()
    for i, s in enumerate(shards):
        arr[i] = RefShard(s["kind"], s["group"], s["rows"], s["offset"], s["k"].shape[0], _d(s["q"]), _d(s["k"]),
                          _d(s["v"]), _d(s["out"]))
    st = C.c_int(0)
    sec = ref().ref_run_shards(arr, len(shards), d, scale, tile_q, tile_kv, threads, C.byref(st))
    if st.value:
        raise OracleError(st.value, "run_shards")
    return sec


_DIST_KIND = {"fixed": 0, "uniform": 1, "lognormal": 2}


def ref_generate_trace(qps, n, pdist, ddist, seed):
    """The reference's generate_trace (serving.hpp:101-118) -> (arrival, prefill, decode) arrays."""
    arr = np.zeros(n)
    pt = np.zeros(n, np.int64)
    dt = np.zeros(n, np.int64)
    st = ref().ref_generate_trace(qps, n, _DIST_KIND[pdist.kind], pdist.a, pdist.b, _DIST_KIND[ddist.kind],
                                  ddist.a, ddist.b, seed, _d(arr), pt.ctypes.data_as(_i64p), dt.ctypes.data_as(_i64p))
    if st:
        raise OracleError(st, "ref_generate_trace")
    return arr, pt, dt


def ref_run_serving_linear(trace, policy, c0, c1):
    """The reference's run_serving (serving.hpp:180-330) with cost c0 + c1 * tokens."""
    n = len(trace)
    arr = np.array([r.arrival_time for r in trace], np.float64)
    pt = np.array([r.prefill_tokens for r in trace], np.int64)
    dt = np.array([r.decode_tokens for r in trace], np.int64)
    cap = 1 << 20
    t0, t1 = np.zeros(cap), np.zeros(cap)
    pr, ptk, nd = (np.zeros(cap, np.int64) for _ in range(3))
    nit = np.zeros(1, np.int64)
    ttft, lat, met = np.zeros(n), np.zeros(n), np.zeros(9)
    i64 = lambda a: a.ctypes.data_as(_i64p)  # noqa: E731
    st = ref().ref_run_serving_linear(n, _d(arr), i64(pt), i64(dt), 0 if policy.kind == "prefill_prioritized" else 1,
                                      policy.chunk_size, policy.max_batch, policy.token_budget, c0, c1, cap,
                                      _d(t0), _d(t1), i64(pr), i64(ptk), i64(nd), i64(nit), _d(ttft), _d(lat), _d(met))
    if st:
        raise OracleError(st, "ref_run_serving_linear")
    k = int(nit[0])
    its = list(zip(t0[:k], t1[:k], pr[:k], ptk[:k], nd[:k]))
    return its, ttft, lat, met
