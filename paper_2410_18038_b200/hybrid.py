"""The GPU operator: one hybrid-batch attention layer through libpod_attn.so.

torch is used only for device memory and the current stream; the compute is
the sm_100a kernels behind the C ABI (pod_attn_run / _serial / _part).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _abi
from ._abi import lib
from .pod import GpuSpec, HybridBatchSpec, InvalidArgument, Plan, PlanOptions, _check


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


@dataclass
class HybridOutputs:
    o_prefill: Optional[torch.Tensor]
    lse_prefill: Optional[torch.Tensor]
    o_decode: Optional[torch.Tensor]
    lse_decode: Optional[torch.Tensor]


def l2_flush(buf: torch.Tensor, stream=None) -> None:
    """pod_attn_l2_flush: zero `buf` (> L2) on the stream, evicting the L2 between timed
    layers without switching the SMs' L1 / shared-memory carve-out (bench utility)."""
    st = stream or torch.cuda.current_stream(buf.device)
    with torch.cuda.device(buf.device):
        _check(lib().pod_attn_l2_flush(_ptr(buf), C.c_int64(buf.numel() * buf.element_size()),
                                       C.c_void_p(st.cuda_stream)), "pod_attn_l2_flush")


class PodAttention:
    """Plan + workspace for one hybrid batch shape; `run` launches the fused kernel."""

    MODES = {"fused": 0, "serial": 1, "prefill": 2, "decode": 3}

    def __init__(self, batch: HybridBatchSpec, gpu: Optional[GpuSpec] = None,
                 options: Optional[PlanOptions] = None, device: int = 0):
        if not torch.cuda.is_available():
            raise RuntimeError("PodAttention needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        self.batch = batch
        self.plan = Plan(batch, gpu or GpuSpec.from_device(device), options)
        self.info = self.plan.info()
        nbytes = max(256, self.plan.workspace_bytes())
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            _check(lib().pod_attn_workspace_init(self.plan.handle, _ptr(self.workspace),
                                                 C.c_void_p(stream.cuda_stream)), "pod_attn_workspace_init")
        self.role_log: Optional[torch.Tensor] = None

    def enable_role_log(self, extra_ints: int = 0) -> torch.Tensor:
        n = int(self.info.num_prefill_ctas + self.info.num_decode_ctas)
        self.role_log = torch.zeros(max(1, n) * 8 + extra_ints, dtype=torch.int32, device=self.device)
        _check(lib().pod_attn_set_role_log(self.plan.handle, _ptr(self.role_log)), "set_role_log")
        return self.role_log

    @property
    def out_dtype(self) -> torch.dtype:
        """Element type of o_prefill / o_decode (PlanOptions.out_dtype); LSE is always fp32."""
        return {_abi.POD_OUT_F32: torch.float32, _abi.POD_OUT_BF16: torch.bfloat16,
                _abi.POD_OUT_F16: torch.float16}[self.plan.options.out_dtype]

    def alloc_outputs(self) -> HybridOutputs:
        s = self.batch.shape
        dev = self.device
        odt = self.out_dtype
        op = lp = od = ld = None
        if self.batch.prefill is not None:
            c = self.batch.prefill.chunk_size
            op = torch.empty(c, s.num_q_heads, s.head_dim, dtype=odt, device=dev)
            lp = torch.empty(c, s.num_q_heads, dtype=torch.float32, device=dev)
        if self.batch.decodes:
            b = len(self.batch.decodes)
            od = torch.empty(b, s.num_q_heads, s.head_dim, dtype=odt, device=dev)
            ld = torch.empty(b, s.num_q_heads, dtype=torch.float32, device=dev)
        return HybridOutputs(op, lp, od, ld)

    def _check_args(self, q_prefill, q_decode, k_pool, v_pool, page_indptr, page_indices, out: HybridOutputs,
                    mode: str) -> None:
        """Shapes, dtypes, contiguity and device of every tensor handed to pod_attn_run*: the
        C ABI takes raw pointers, so a mismatch here would be silently misread by the kernels."""
        b, s = self.batch, self.batch.shape
        kv_dt = torch.float16 if b.dtype == _abi.POD_DTYPE_FP16 else torch.bfloat16
        m = self.MODES[mode]
        need_p = b.prefill is not None and m != 3
        need_d = bool(b.decodes) and m != 2

        def t(x, name, dtype, shape=None):
            if x is None:
                raise InvalidArgument(f"{name} is required for this batch")
            if x.device != self.device:
                raise InvalidArgument(f"{name} is on {x.device}, the plan runs on {self.device}")
            if x.dtype != dtype:
                raise InvalidArgument(f"{name} must be {dtype}, got {x.dtype}")
            if not x.is_contiguous():
                raise InvalidArgument(f"{name} must be contiguous")
            if shape is not None and tuple(x.shape) != tuple(shape):
                raise InvalidArgument(f"{name} has shape {tuple(x.shape)}, expected {tuple(shape)}")

        if k_pool.dim() != 4 or k_pool.shape != v_pool.shape:
            raise InvalidArgument("k_pool / v_pool must be equal 4-D pools")
        ps = b.page_size
        pool = ((k_pool.shape[0], s.num_kv_heads, ps, s.head_dim) if b.kv_layout == _abi.POD_KV_HND
                else (k_pool.shape[0], ps, s.num_kv_heads, s.head_dim))
        t(k_pool, "k_pool", kv_dt, pool)
        t(v_pool, "v_pool", kv_dt, pool)
        nreq = (1 if b.prefill is not None else 0) + len(b.decodes)
        t(page_indptr, "page_indptr", torch.int32, (nreq + 1,))
        t(page_indices, "page_indices", torch.int32)
        odt = self.out_dtype
        if need_p:
            c = b.prefill.chunk_size
            t(q_prefill, "q_prefill", kv_dt, (c, s.num_q_heads, s.head_dim))
            t(out.o_prefill, "o_prefill", odt, (c, s.num_q_heads, s.head_dim))
            t(out.lse_prefill, "lse_prefill", torch.float32, (c, s.num_q_heads))
        if need_d:
            nb = len(b.decodes)
            t(q_decode, "q_decode", kv_dt, (nb, s.num_q_heads, s.head_dim))
            t(out.o_decode, "o_decode", odt, (nb, s.num_q_heads, s.head_dim))
            t(out.lse_decode, "lse_decode", torch.float32, (nb, s.num_q_heads))

    def run(self, q_prefill, q_decode, k_pool, v_pool, page_indptr, page_indices,
            out: Optional[HybridOutputs] = None, mode: str = "fused", stream=None) -> HybridOutputs:
        out = out or self.alloc_outputs()
        self._check_args(q_prefill, q_decode, k_pool, v_pool, page_indptr, page_indices, out, mode)
        with torch.cuda.device(self.device):
            return self._launch(q_prefill, q_decode, k_pool, v_pool, page_indptr, page_indices, out, mode, stream)

    def _launch(self, q_prefill, q_decode, k_pool, v_pool, page_indptr, page_indices, out, mode, stream):
        st = stream or torch.cuda.current_stream(self.device)
        num_pages = k_pool.shape[0]
        args = (_ptr(q_prefill), _ptr(q_decode), _ptr(k_pool), _ptr(v_pool), C.c_int64(num_pages),
                _ptr(page_indptr), _ptr(page_indices), _ptr(out.o_prefill), _ptr(out.lse_prefill),
                _ptr(out.o_decode), _ptr(out.lse_decode), _ptr(self.workspace), C.c_void_p(st.cuda_stream))
        m = self.MODES[mode]
        L = lib()
        if m == 0:
            _check(L.pod_attn_run(self.plan.handle, *args), "pod_attn_run")
        elif m == 1:
            _check(L.pod_attn_run_serial(self.plan.handle, *args), "pod_attn_run_serial")
        else:
            _check(L.pod_attn_run_part(self.plan.handle, m - 2, *args), "pod_attn_run_part")
        return out

    def append_kv(self, k_new_prefill, v_new_prefill, k_new_decode, v_new_decode, k_pool, v_pool, page_indptr,
                  page_indices, stream=None) -> None:
        """pod_attn_append_kv: scatter the batch's new K/V rows ([chunk][Hkv][d] and
        [B][Hkv][d], pool dtype) into their page slots (before run())."""
        st = stream or torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            self._append(k_new_prefill, v_new_prefill, k_new_decode, v_new_decode, k_pool, v_pool, page_indptr,
                         page_indices, st)

    def _append(self, k_new_prefill, v_new_prefill, k_new_decode, v_new_decode, k_pool, v_pool, page_indptr,
                page_indices, st) -> None:
        _check(lib().pod_attn_append_kv(self.plan.handle, _ptr(k_new_prefill), _ptr(v_new_prefill), _ptr(k_new_decode),
                                        _ptr(v_new_decode), _ptr(k_pool), _ptr(v_pool), C.c_int64(k_pool.shape[0]),
                                        _ptr(page_indptr), _ptr(page_indices), _ptr(self.workspace),
                                        C.c_void_p(st.cuda_stream)), "pod_attn_append_kv")

    def gather_probe(self, pool: torch.Tensor, page_indptr, page_indices, req: int, ctx: int) -> torch.Tensor:
        s = self.batch.shape
        out = torch.empty(ctx, s.num_kv_heads, s.head_dim, dtype=torch.int16, device=self.device)
        st = torch.cuda.current_stream(self.device)
        _check(lib().pod_attn_gather_probe(self.plan.handle, _ptr(pool), C.c_int64(pool.shape[0]), _ptr(page_indptr),
                                           _ptr(page_indices), req, ctx, _ptr(out), C.c_void_p(st.cuda_stream)),
               "gather_probe")
        return out
