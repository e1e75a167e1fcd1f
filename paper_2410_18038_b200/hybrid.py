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
from .pod import GpuSpec, HybridBatchSpec, Plan, PlanOptions, _check


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


@dataclass
class HybridOutputs:
    o_prefill: Optional[torch.Tensor]
    lse_prefill: Optional[torch.Tensor]
    o_decode: Optional[torch.Tensor]
    lse_decode: Optional[torch.Tensor]


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
        _check(lib().pod_attn_workspace_init(self.plan.handle, _ptr(self.workspace), C.c_void_p(stream.cuda_stream)),
               "pod_attn_workspace_init")
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

    def run(self, q_prefill, q_decode, k_pool, v_pool, page_indptr, page_indices,
            out: Optional[HybridOutputs] = None, mode: str = "fused", stream=None) -> HybridOutputs:
        out = out or self.alloc_outputs()
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
