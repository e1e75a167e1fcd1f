"""Measured kernel selection for one hybrid-batch shape.

The reference picks its configuration by searching its GPU simulator:
`best_fused_makespan` (gpu_sim.hpp:802-816) tries {2, 4} CTAs per SM x {50:50,
proportional} and keeps the smallest simulated makespan.  POD_POLICY_AUTO replaces
that with rules measured on B200 (pod_plan.cpp); `tune_options` is the search
itself, on the hardware: it plans the batch with every candidate (the two POD
kernels, both pair-engine tile widths, split caps), runs each on synthetic inputs of
the batch's shape with the L2 flushed between runs, and returns the fastest options
and the timing table.  `TunedOptions` memoises the choice per batch signature (the
serving loop's bucketed shapes), like the reference's IterationCostModel memo
(serving.hpp:128-160).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

from . import _abi
from .pod import HybridBatchSpec, PlanOptions, Unsupported


def default_candidates(batch: HybridBatchSpec) -> List[Tuple[str, PlanOptions]]:
    c = [("auto", PlanOptions())]
    if batch.prefill is not None:
        c += [("warpspec/32-key", PlanOptions(policy=_abi.POD_POLICY_WARPSPEC, prefill_tile_keys=32)),
              ("warpspec/64-key", PlanOptions(policy=_abi.POD_POLICY_WARPSPEC, prefill_tile_keys=64,
                                              prefill_s_buffers=1)),
              ("warpspec/64-key/double-S", PlanOptions(policy=_abi.POD_POLICY_WARPSPEC, prefill_tile_keys=64,
                                                       prefill_s_buffers=2))]
    for cap in (0, 2, 4):
        c.append((f"complement/cap{cap or 'auto'}", PlanOptions(policy=_abi.POD_POLICY_COMPLEMENT, split_wave_cap=cap)))
    return c


def tune_options(batch: HybridBatchSpec, device: int = 0, candidates: Optional[Sequence[Tuple[str, PlanOptions]]] = None,
                 reps: int = 5, warmup: int = 2, flush_bytes: int = 512 << 20, workload=None):
    """Times every candidate's fused layer on this batch shape; returns (best PlanOptions,
    [(name, median us) ...] sorted fastest first).  Candidates the planner rejects for
    the shape (Unsupported) are skipped."""
    import torch

    from .hybrid import PodAttention, l2_flush
    from .workload import build_workload

    dev = torch.device("cuda", device)
    wl = workload or build_workload(batch, device=dev)
    flush = torch.empty(flush_bytes, dtype=torch.uint8, device=dev)
    table = []
    best = None
    for name, opts in candidates or default_candidates(batch):
        try:
            op = PodAttention(batch, options=opts, device=device)
        except Unsupported:
            continue
        out = op.alloc_outputs()

        def step():
            op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, out=out)

        for _ in range(warmup):
            step()
        ts = []
        for _ in range(reps):
            l2_flush(flush)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000.0)
        us = sorted(ts)[len(ts) // 2]
        table.append((name, round(us, 2)))
        if best is None or us < best[1]:
            best = (opts, us)
        del op, out
    table.sort(key=lambda x: x[1])
    return best[0], table


class TunedOptions:
    """Per-shape memo of tune_options: `options(batch)` returns the fastest PlanOptions
    measured for the batch's bucketed signature (decode contexts and the prefill offset
    rounded up to `bucket` tokens)."""

    def __init__(self, device: int = 0, bucket: int = 256, reps: int = 5):
        self.device, self.bucket, self.reps = device, bucket, reps
        self.memo: Dict[Tuple, PlanOptions] = {}
        self.tables: Dict[Tuple, list] = {}

    def _round(self, x: int) -> int:
        return ((x + self.bucket - 1) // self.bucket) * self.bucket

    def signature(self, batch: HybridBatchSpec) -> Tuple:
        s = batch.shape
        pf = batch.prefill
        p = (pf.chunk_size, self._round(pf.position_offset)) if pf is not None else None
        return (s.num_q_heads, s.num_kv_heads, p, tuple(sorted(self._round(d.context_len) for d in batch.decodes)))

    def options(self, batch: HybridBatchSpec) -> PlanOptions:
        key = self.signature(batch)
        if key not in self.memo:
            self.memo[key], self.tables[key] = tune_options(batch, self.device, reps=self.reps)
        return self.memo[key]
