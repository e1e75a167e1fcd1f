"""Synthetic hybrid batches for the bench and the parity tests.

Values follow the reference tests' recipe (proj/tests/test_attention.cpp:69-72):
x = Rng.next_double() * 2 - 1 with the splitmix64 Rng of rng.hpp:11-47, then
rounded to bf16 (via fp32, RNE).  The Rng stream is evaluated position-wise
(splitmix64's state after i draws is seed + (i+1) * golden), so any slice can
be regenerated on the GPU or the CPU without materialising the rest.

Stream assignment (seeds per SURVEY.md 8(d)):
  Rng(42): prefill Q [chunk][Hq][d], then decode Q [B][Hq][d]   (x `q_scale`)
  Rng(43): K of every request ([ctx_i][Hkv][d], request order), then V likewise
  Rng(44): Fisher-Yates permutation of the physical pages (block tables)
Request 0 is the prefill (its cache holds position_offset + chunk tokens),
then the decodes.  Pool layout HND [num_pages][Hkv][page_size][d]; padding
slots of a request's last page hold the constant `pad_value`.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import torch

from .pod import DecodeSpec, HybridBatchSpec, ModelShape, PrefillSpec

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def _s64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= 1 << 63 else x


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix_u64(seed: int, positions: torch.Tensor) -> torch.Tensor:
    """next_u64() after `positions` previous draws (rng.hpp:15-20), as int64 bit patterns."""
    z = positions.to(torch.int64) + 1
    z = z * _s64(_GOLDEN) + _s64(seed)
    z = (z ^ _srl(z, 30)) * _s64(_M1)
    z = (z ^ _srl(z, 27)) * _s64(_M2)
    return z ^ _srl(z, 31)


def rng_doubles(seed: int, start: int, n: int, device="cpu") -> torch.Tensor:
    """next_double() (rng.hpp:23) for stream positions [start, start + n)."""
    pos = torch.arange(start, start + n, dtype=torch.int64, device=device)
    return _srl(splitmix_u64(seed, pos), 11).to(torch.float64) * (2.0 ** -53)


def rng_values(seed: int, start: int, n: int, device="cpu", scale: float = 1.0,
               dtype=torch.bfloat16) -> torch.Tensor:
    """x = next_double()*2-1 (times `scale`), rounded to `dtype`; generated in chunks."""
    out = torch.empty(n, dtype=dtype, device=device)
    step = 1 << 26
    for s in range(0, n, step):
        m = min(step, n - s)
        x = rng_doubles(seed, start + s, m, device) * 2.0 - 1.0
        out[s:s + m] = (x * scale).to(torch.float32).to(dtype)
    return out


def rng_permutation(seed: int, n: int) -> List[int]:
    """Fisher-Yates with next_u64() % i (the reference's shuffle, gpu_sim.hpp:414-418)."""
    draws = splitmix_u64(seed, torch.arange(0, max(0, n - 1), dtype=torch.int64)).tolist()
    perm = list(range(n))
    for j, i in enumerate(range(n, 1, -1)):
        r = draws[j] & ((1 << 64) - 1)
        k = r % i
        perm[i - 1], perm[k] = perm[k], perm[i - 1]
    return perm


@dataclass
class HybridWorkload:
    batch: HybridBatchSpec
    q_prefill: Optional[torch.Tensor]
    q_decode: Optional[torch.Tensor]
    k_pool: torch.Tensor
    v_pool: torch.Tensor
    page_indptr: torch.Tensor
    page_indices: torch.Tensor
    kv_lens: List[int] = field(default_factory=list)     # tokens in each request's cache
    kv_offsets: List[int] = field(default_factory=list)  # element offset of request i in the K (or V) stream
    kv_total: int = 0
    q_scale: float = 1.0
    seed_q: int = 42
    seed_kv: int = 43
    seed_pages: int = 44

    # -- regenerate reference (contiguous, unpaged) inputs on the CPU ---------
    def request_cache(self, req: int, which: str, head: Optional[int] = None) -> torch.Tensor:
        """Contiguous cache [ctx][Hkv][d] (or [ctx][d] for one head) as float64,
        regenerated from the Rng: the reference's KVCacheT layout (attention.hpp:36-38)."""
        s = self.batch.shape
        ctx = self.kv_lens[req]
        base = self.kv_offsets[req] + (self.kv_total if which == "v" else 0)
        if head is None:
            x = rng_values(self.seed_kv, base, ctx * s.num_kv_heads * s.head_dim)
            return x.to(torch.float64).view(ctx, s.num_kv_heads, s.head_dim)
        pos = (torch.arange(ctx, dtype=torch.int64)[:, None] * (s.num_kv_heads * s.head_dim)
               + head * s.head_dim + torch.arange(s.head_dim, dtype=torch.int64)[None, :]).reshape(-1) + base
        u = _srl(splitmix_u64(self.seed_kv, pos), 11).to(torch.float64) * (2.0 ** -53)
        return (u * 2.0 - 1.0).to(torch.float32).to(torch.bfloat16).to(torch.float64).view(ctx, s.head_dim)

    def prefill_q(self) -> torch.Tensor:
        s = self.batch.shape
        c = self.batch.prefill.chunk_size
        return rng_values(self.seed_q, 0, c * s.num_q_heads * s.head_dim, scale=self.q_scale).to(
            torch.float64).view(c, s.num_q_heads, s.head_dim)

    def decode_q(self) -> torch.Tensor:
        s = self.batch.shape
        n0 = self.batch.prefill.chunk_size * s.num_q_heads * s.head_dim if self.batch.prefill else 0
        b = len(self.batch.decodes)
        return rng_values(self.seed_q, n0, b * s.num_q_heads * s.head_dim, scale=self.q_scale).to(
            torch.float64).view(b, s.num_q_heads, s.head_dim)


def make_batch(shape: ModelShape, chunk: int = 0, offset: int = 0, prompt: Optional[int] = None,
               decode_ctx: Optional[List[int]] = None, page_size: int = 16) -> HybridBatchSpec:
    pf = None
    if chunk > 0:
        pf = PrefillSpec(chunk, prompt if prompt is not None else offset + chunk, offset)
    return HybridBatchSpec(prefill=pf, decodes=[DecodeSpec(c) for c in (decode_ctx or [])], shape=shape,
                           page_size=page_size)


def build_workload(batch: HybridBatchSpec, device="cpu", q_scale: float = 1.0, pad_value: float = 0.0,
                   extra_pages: int = 0, seed_q: int = 42, seed_kv: int = 43, seed_pages: int = 44,
                   dtype=torch.bfloat16) -> HybridWorkload:
    s = batch.shape
    ps = batch.page_size
    hkv, d = s.num_kv_heads, s.head_dim
    kv_lens: List[int] = []
    if batch.prefill is not None:
        kv_lens.append(batch.prefill.position_offset + batch.prefill.chunk_size)
    kv_lens += [dd.context_len for dd in batch.decodes]
    pages = [(n + ps - 1) // ps for n in kv_lens]
    total_pages = sum(pages) + extra_pages
    perm = rng_permutation(seed_pages, total_pages)
    indptr = [0]
    for n in pages:
        indptr.append(indptr[-1] + n)
    indices = [perm[i] for i in range(indptr[-1])]
    offsets, off = [], 0
    for n in kv_lens:
        offsets.append(off)
        off += n * hkv * d
    kv_total = off

    q_prefill = q_decode = None
    nq0 = 0
    if batch.prefill is not None:
        nq0 = batch.prefill.chunk_size * s.num_q_heads * d
        q_prefill = rng_values(seed_q, 0, nq0, device, q_scale, dtype).view(batch.prefill.chunk_size,
                                                                            s.num_q_heads, d)
    if batch.decodes:
        nb = len(batch.decodes) * s.num_q_heads * d
        q_decode = rng_values(seed_q, nq0, nb, device, q_scale, dtype).view(len(batch.decodes), s.num_q_heads, d)

    pools = []
    for which in (0, 1):
        pool = torch.full((total_pages, hkv, ps, d), pad_value, dtype=dtype, device=device)
        for r, n in enumerate(kv_lens):
            x = rng_values(seed_kv, offsets[r] + which * kv_total, n * hkv * d, device, 1.0, dtype).view(n, hkv, d)
            npg = pages[r]
            if npg * ps != n:
                padded = torch.full((npg * ps, hkv, d), pad_value, dtype=dtype, device=device)
                padded[:n] = x
                x = padded
            phys = torch.tensor(indices[indptr[r]:indptr[r + 1]], dtype=torch.int64, device=device)
            pool[phys] = x.view(npg, ps, hkv, d).permute(0, 2, 1, 3)
        pools.append(pool)
    return HybridWorkload(batch, q_prefill, q_decode, pools[0], pools[1],
                          torch.tensor(indptr, dtype=torch.int32, device=device),
                          torch.tensor(indices if indices else [0], dtype=torch.int32, device=device),
                          kv_lens, offsets, kv_total, q_scale, seed_q, seed_kv, seed_pages)


class Rng:
    """Sequential splitmix64 (rng.hpp:11-47) with exact integer arithmetic, for
    reproducing the reference tests' interleaved draws (next_long, fills)."""

    def __init__(self, seed: int):
        self.state = seed & ((1 << 64) - 1)
        self.pos = 0  # draws so far (the vectorised generator's position)
        self.seed = seed

    def next_u64(self) -> int:
        self.state = (self.state + _GOLDEN) & ((1 << 64) - 1)
        z = self.state
        z = ((z ^ (z >> 30)) * _M1) & ((1 << 64) - 1)
        z = ((z ^ (z >> 27)) * _M2) & ((1 << 64) - 1)
        self.pos += 1
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def next_long(self, lo: int, hi: int) -> int:
        return lo + self.next_u64() % (hi - lo + 1)

    def fill_uniform(self, n: int):
        """n draws of next_double()*2-1 as float64 (vectorised), advancing the stream."""
        x = rng_doubles(self.seed, self.pos, n) * 2.0 - 1.0
        self.pos += n
        self.state = (self.seed + self.pos * _GOLDEN) & ((1 << 64) - 1)
        return x
