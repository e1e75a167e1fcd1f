"""Serving loop over the B200 POD kernels.

The reference's request-level simulator (serving.hpp) builds one HybridBatchSpec
per iteration -- a prefill chunk riding along with every active decode
(chunked-prefill hybrid batching) or whole-prompt prefills that pause decodes
(prefill-prioritised) -- and charges each iteration `w_fixed + w_tok * tokens +
attention_cost(batch)`, where the reference's attention cost comes from its GPU
*simulator* (serving.hpp:123-169).  This module is that caller, restated
(`run_serving` follows serving.hpp:180-330 step by step; the loop is pinned
against the compiled reference in tests/test_serving.py), with the attention term
**measured** on the B200: `MeasuredIterationCost` plans and runs the batch
through `pod_attn_run` (fused) or `pod_attn_run_serial` and times it with CUDA
events, so the kernel's speed-up turns into TTFT / TBT numbers.

Times are in microseconds when the measured cost is used.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from .pod import DecodeSpec, HybridBatchSpec, ModelShape, PlanOptions, PrefillSpec
from .workload import Rng


@dataclass
class Request:  # serving.hpp:22-26
    arrival_time: float = 0.0
    prefill_tokens: int = 1
    decode_tokens: int = 1


@dataclass
class SchedulerPolicy:  # serving.hpp:28-52
    kind: str = "chunked_hybrid"  # or "prefill_prioritized"
    chunk_size: int = 1024
    max_batch: int = 256
    token_budget: int = 4096

    @staticmethod
    def prefill_prioritized() -> "SchedulerPolicy":
        return SchedulerPolicy("prefill_prioritized", 0, 256, 0)

    @staticmethod
    def chunked_hybrid(chunk: int, max_batch: int = 256, token_budget: int = 1 << 20) -> "SchedulerPolicy":
        return SchedulerPolicy("chunked_hybrid", chunk, max_batch, token_budget)

    def validate(self) -> None:
        if self.kind == "chunked_hybrid":
            if self.chunk_size < 1:
                raise ValueError("SchedulerPolicy: chunk_size < 1")
            if self.token_budget < self.chunk_size:
                raise ValueError("SchedulerPolicy: token_budget < chunk_size")


@dataclass
class IterationRecord:  # serving.hpp:54-60
    t_start: float = 0.0
    t_end: float = 0.0
    prefill_request: int = -1
    prefill_tokens: int = 0
    decode_requests: int = 0


@dataclass
class Metrics:  # serving.hpp:62-68
    ttft_p50: float = 0.0
    ttft_p99: float = 0.0
    tbt_p50: float = 0.0
    tbt_p99: float = 0.0
    latency_p50: float = 0.0
    latency_p99: float = 0.0
    stall_pct_at: List[Tuple[float, float]] = field(default_factory=list)
    throughput: float = 0.0


@dataclass
class ServingResult:  # serving.hpp:171-176
    metrics: Metrics
    iterations: List[IterationRecord]
    ttft: List[float]
    latency: List[float]
    tbt: List[List[float]]


def percentile(samples: Sequence[float], p: float) -> float:
    """Nearest rank: the ceil(p/100 * n)-th smallest (1-based) (serving.hpp:72-80)."""
    if not samples:
        raise ValueError("percentile: empty sample set")
    if p < 0 or p > 100:
        raise ValueError("percentile: p out of range")
    s = sorted(samples)
    n = len(s)
    rank = min(max(int(math.ceil(p / 100.0 * n)), 1), n)
    return s[rank - 1]


@dataclass
class TokenDist:  # serving.hpp:82-97
    kind: str = "fixed"  # fixed | uniform | lognormal
    a: float = 1024.0
    b: float = 0.0

    def sample(self, rng: Rng) -> int:
        if self.kind == "fixed":
            x = self.a
        elif self.kind == "uniform":
            x = self.a + rng.next_double() * (self.b - self.a)
        else:  # Box-Muller lognormal (rng.hpp:36-43)
            u1 = rng.next_double()
            u2 = rng.next_double()
            while u1 <= 0.0:
                u1 = rng.next_double()
            z = math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)
            x = math.exp(self.a + self.b * z)
        return max(1, _llround(x))


def _llround(x: float) -> int:
    """std::llround: half away from zero."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def generate_trace(qps: float, n: int, prefill_dist: TokenDist, decode_dist: TokenDist,
                   seed: int) -> List[Request]:
    """Poisson arrivals at rate qps (serving.hpp:101-118; exponential gaps rng.hpp:31-34)."""
    if not qps > 0:
        raise ValueError("generate_trace: qps must be positive")
    rng = Rng(seed)
    t = 0.0
    out = []
    for _ in range(n):
        u = rng.next_double()
        t += -math.log1p(-u) / qps
        out.append(Request(t, prefill_dist.sample(rng), decode_dist.sample(rng)))
    return out


def run_serving(trace: Sequence[Request], policy: SchedulerPolicy,
                iteration_cost: Callable[[HybridBatchSpec, bool], float], fused: bool, shape: ModelShape,
                stall_thresholds: Sequence[float] = (200.0, 500.0)) -> ServingResult:
    """The reference's iteration loop (serving.hpp:180-330)."""
    if not trace:
        raise ValueError("run_serving: empty trace")
    policy.validate()
    for i in range(1, len(trace)):
        if trace[i].arrival_time < trace[i - 1].arrival_time:
            raise ValueError("run_serving: trace not sorted by arrival")
    n = len(trace)
    prefill_done = [0] * n
    generated = [0] * n
    last_token = [0.0] * n
    ttft = [0.0] * n
    latency = [0.0] * n
    tbt: List[List[float]] = [[] for _ in range(n)]
    iterations: List[IterationRecord] = []
    waiting: List[int] = []
    decoding: List[int] = []
    mid_prefill = -1
    next_arrival = 0
    completed = 0
    now = 0.0

    def admit(t: float) -> None:
        nonlocal next_arrival
        while next_arrival < n and trace[next_arrival].arrival_time <= t:
            waiting.append(next_arrival)
            next_arrival += 1

    admit(0.0)
    while completed < n:
        if not waiting and not decoding and mid_prefill < 0:
            now = max(now, trace[next_arrival].arrival_time)
            admit(now)
            continue
        prefill = None
        prefill_req = -1
        chunk = 0
        decode_advances = False
        if policy.kind == "prefill_prioritized":
            if waiting:
                prefill_req = waiting.pop(0)
                chunk = trace[prefill_req].prefill_tokens
                prefill = PrefillSpec(chunk, trace[prefill_req].prefill_tokens, 0)
            else:
                decode_advances = True
        else:
            if mid_prefill < 0 and waiting and len(decoding) + 1 <= policy.max_batch:
                mid_prefill = waiting.pop(0)
            if mid_prefill >= 0:
                remaining = trace[mid_prefill].prefill_tokens - prefill_done[mid_prefill]
                budget = policy.token_budget - len(decoding)
                chunk = min(policy.chunk_size, remaining, max(1, budget))
                prefill_req = mid_prefill
                prefill = PrefillSpec(chunk, trace[prefill_req].prefill_tokens, prefill_done[prefill_req])
            decode_advances = True
        decodes = ([DecodeSpec(trace[i].prefill_tokens + generated[i]) for i in decoding]
                   if decode_advances else [])
        batch = HybridBatchSpec(prefill=prefill, decodes=decodes, shape=shape)
        cost = iteration_cost(batch, fused)
        t_end = now + cost
        iterations.append(IterationRecord(now, t_end, prefill_req, chunk, len(decoding) if decode_advances else 0))
        if decode_advances:
            i = 0
            while i < len(decoding):
                rid = decoding[i]
                tbt[rid].append(t_end - last_token[rid])
                last_token[rid] = t_end
                generated[rid] += 1
                if generated[rid] >= trace[rid].decode_tokens:
                    latency[rid] = t_end - trace[rid].arrival_time
                    decoding.pop(i)
                    completed += 1
                else:
                    i += 1
        if prefill_req >= 0:
            prefill_done[prefill_req] += chunk
            if prefill_done[prefill_req] >= trace[prefill_req].prefill_tokens:
                ttft[prefill_req] = t_end - trace[prefill_req].arrival_time
                last_token[prefill_req] = t_end
                if prefill_req == mid_prefill:
                    mid_prefill = -1
                decoding.append(prefill_req)
        now = t_end
        admit(now)
    all_tbt = [x for v in tbt for x in v]
    m = Metrics(ttft_p50=percentile(ttft, 50), ttft_p99=percentile(ttft, 99),
                latency_p50=percentile(latency, 50), latency_p99=percentile(latency, 99))
    if all_tbt:
        m.tbt_p50 = percentile(all_tbt, 50)
        m.tbt_p99 = percentile(all_tbt, 99)
    for thr in stall_thresholds:
        stalled = sum(1 for v in tbt if any(x > thr for x in v))
        m.stall_pct_at.append((thr, stalled / n))
    m.throughput = n / now if now > 0 else 0.0
    return ServingResult(m, iterations, ttft, latency, tbt)


class MeasuredIterationCost:
    """Iteration cost `w_fixed + w_tok * tokens + attention_us`, the attention term
    measured on the GPU through pod_attn_run (fused) / pod_attn_run_serial: the
    batch is planned with the default options, run `repeats` times on synthetic
    inputs over one shared paged pool (values do not affect the time) and the
    median CUDA-event time is taken (times `layers`).  Memoised per batch signature like the
    reference's IterationCostModel (serving.hpp:128-160); decode contexts and the
    prefill offset are rounded up to `bucket` tokens to bound the distinct shapes."""

    def __init__(self, shape: ModelShape, w_fixed: float = 0.0, w_tok: float = 0.0, device: int = 0,
                 bucket: int = 256, repeats: int = 5, options: Optional[PlanOptions] = None, layers: int = 1):
        import torch

        self.torch = torch
        self.shape = shape
        self.w_fixed, self.w_tok = w_fixed, w_tok
        self.device = torch.device("cuda", device)
        self.bucket = bucket
        self.repeats = repeats
        self.options = options
        self.layers = layers  # attention layers per iteration (the measured layer time x layers)
        self.memo: Dict[Tuple, float] = {}
        self._pool_pages = 0
        self.k_pool = self.v_pool = None
        self.measurements = 0

    def _round(self, x: int) -> int:
        return ((x + self.bucket - 1) // self.bucket) * self.bucket

    def _signature(self, batch: HybridBatchSpec, fused: bool) -> Tuple:
        pf = batch.prefill
        p = (pf.chunk_size, self._round(pf.position_offset)) if pf is not None else None
        return (fused, p, tuple(sorted(self._round(d.context_len) for d in batch.decodes)))

    def _ensure_pool(self, pages: int) -> None:
        torch = self.torch
        if pages <= self._pool_pages:
            return
        pages = max(pages, int(self._pool_pages * 1.5))
        s = self.shape
        shp = (pages, s.num_kv_heads, 16, s.head_dim)
        g = torch.Generator(device=self.device).manual_seed(43)
        self.k_pool = (torch.rand(shp, generator=g, device=self.device, dtype=torch.float32) * 2 - 1).to(torch.bfloat16)
        self.v_pool = (torch.rand(shp, generator=g, device=self.device, dtype=torch.float32) * 2 - 1).to(torch.bfloat16)
        self._pool_pages = pages

    def attention_us(self, batch: HybridBatchSpec, fused: bool) -> float:
        key = self._signature(batch, fused)
        if key in self.memo:
            return self.memo[key]
        torch = self.torch
        from .hybrid import PodAttention

        s = self.shape
        pf = batch.prefill
        # measured shape: bucketed contexts (same chunk)
        mpf = None
        ctxs = []
        if pf is not None:
            off = self._round(pf.position_offset)
            mpf = PrefillSpec(pf.chunk_size, off + pf.chunk_size, off)
            ctxs.append(off + pf.chunk_size)
        decs = [DecodeSpec(self._round(d.context_len)) for d in batch.decodes]
        ctxs += [d.context_len for d in decs]
        mb = HybridBatchSpec(prefill=mpf, decodes=decs, shape=s)
        pages_per = [(c + 15) // 16 for c in ctxs]
        total = sum(pages_per)
        self._ensure_pool(total)
        g = torch.Generator(device="cpu").manual_seed(44 + total)
        perm = torch.randperm(self._pool_pages, generator=g)[:total].to(torch.int32)
        indptr = torch.tensor([0] + list(_cumsum(pages_per)), dtype=torch.int32)
        q_p = torch.rand(pf.chunk_size, s.num_q_heads, s.head_dim, device=self.device).to(torch.bfloat16) \
            if pf is not None else None
        q_d = torch.rand(len(decs), s.num_q_heads, s.head_dim, device=self.device).to(torch.bfloat16) \
            if decs else None
        op = PodAttention(mb, options=self.options, device=self.device.index or 0)
        out = op.alloc_outputs()
        ip, ix = indptr.to(self.device), perm.to(self.device)
        mode = "fused" if fused else "serial"
        for _ in range(2):
            op.run(q_p, q_d, self.k_pool, self.v_pool, ip, ix, out=out, mode=mode)
        times = []
        for _ in range(self.repeats):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op.run(q_p, q_d, self.k_pool, self.v_pool, ip, ix, out=out, mode=mode)
            e1.record()
            times.append((e0, e1))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in times)
        us = ms[len(ms) // 2] * 1000.0
        op.plan.close()
        self.memo[key] = us
        self.measurements += 1
        return us

    def __call__(self, batch: HybridBatchSpec, fused: bool) -> float:
        if batch.prefill is None and not batch.decodes:
            raise ValueError("iteration_cost: empty batch")
        tokens = (batch.prefill.chunk_size if batch.prefill is not None else 0) + len(batch.decodes)
        return self.w_fixed + self.w_tok * tokens + self.layers * self.attention_us(batch, fused)


def _cumsum(xs):
    t = 0
    for x in xs:
        t += x
        yield t
