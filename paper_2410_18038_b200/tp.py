"""KV-head-group tensor parallelism for the hybrid-batch layer.

Rank t of T owns KV heads [t*Hkv/T, (t+1)*Hkv/T) and their `group` query heads,
so attention needs no exchange; one all-gather of the per-rank outputs
[tokens][Hq/T][d] (+ LSE [tokens][Hq/T]) assembles the layer output
[tokens][Hq][d].

The kernel writes straight into the all-gather send buffer: `GatherBuffers`
carves o_prefill / o_decode / lse_prefill / lse_decode out of ONE byte buffer
([O: tokens x Hq/T x d of the output dtype][LSE: tokens x Hq/T fp32]), so the
step is kernel -> one all-gather, with no copy in between, and the consumer reads
the rank-major receive buffer through `assemble_layer` views.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Tuple

import torch

from .pod import ModelShape


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_head_begin: int
    kv_head_end: int
    q_head_begin: int
    q_head_end: int
    shape: ModelShape  # per-rank shape (Hq/T, Hkv/T, d, scale)


def shard_heads(shape: ModelShape, rank: int, world: int) -> HeadShard:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if shape.num_kv_heads % world:
        raise ValueError(f"num_kv_heads={shape.num_kv_heads} is not divisible by TP={world}")
    hkv = shape.num_kv_heads // world
    g = shape.group_size()
    kb = rank * hkv
    return HeadShard(rank, world, kb, kb + hkv, kb * g, (kb + hkv) * g,
                     ModelShape(hkv * g, hkv, shape.head_dim, shape.scale))


def slice_heads(x: torch.Tensor, shard: HeadShard, kv: bool) -> torch.Tensor:
    """Selects this rank's heads from a [..., H, d] tensor (H = Hkv if kv else Hq)."""
    b, e = (shard.kv_head_begin, shard.kv_head_end) if kv else (shard.q_head_begin, shard.q_head_end)
    return x[..., b:e, :]


def shard_workload(wl, shard: HeadShard):
    """This rank's slice of one full-layer workload (workload.HybridWorkload): the same
    requests and block tables, Q restricted to the rank's q heads and the paged pools to
    its KV heads (HND [pages][Hkv][page][d] -> [pages][Hkv/T][page][d]), contiguous."""
    if wl.batch.kv_layout != 0:
        raise ValueError("shard_workload: HND pools only")
    batch = replace(wl.batch, shape=shard.shape)
    kb, ke = shard.kv_head_begin, shard.kv_head_end
    qp = slice_heads(wl.q_prefill, shard, kv=False).contiguous() if wl.q_prefill is not None else None
    qd = slice_heads(wl.q_decode, shard, kv=False).contiguous() if wl.q_decode is not None else None
    return replace(wl, batch=batch, q_prefill=qp, q_decode=qd, k_pool=wl.k_pool[:, kb:ke].contiguous(),
                   v_pool=wl.v_pool[:, kb:ke].contiguous())


@dataclass
class GatherBuffers:
    send: torch.Tensor            # uint8 [rank_bytes]: O then LSE of this rank
    recv: torch.Tensor            # uint8 [world * rank_bytes], rank-major
    outputs: object               # hybrid.HybridOutputs: views into `send`
    tokens: int
    chunk: int
    hq_rank: int
    head_dim: int
    out_dtype: torch.dtype
    world: int


def gather_buffers(batch, world: int, out_dtype: torch.dtype, device) -> GatherBuffers:
    """One send buffer per rank; the kernel's four outputs are views into it."""
    from .hybrid import HybridOutputs

    s = batch.shape
    chunk = batch.prefill.chunk_size if batch.prefill is not None else 0
    nb = len(batch.decodes)
    tokens, hq, d = chunk + nb, s.num_q_heads, s.head_dim
    esz = torch.empty((), dtype=out_dtype).element_size()
    o_bytes = tokens * hq * d * esz
    o_pad = (o_bytes + 15) // 16 * 16
    rank_bytes = o_pad + tokens * hq * 4
    send = torch.zeros(rank_bytes, dtype=torch.uint8, device=device)
    o = send[:o_bytes].view(out_dtype).view(tokens, hq, d)
    lse = send[o_pad:].view(torch.float32).view(tokens, hq)
    outs = HybridOutputs(o[:chunk] if chunk else None, lse[:chunk] if chunk else None,
                         o[chunk:] if nb else None, lse[chunk:] if nb else None)
    recv = torch.empty(world * rank_bytes, dtype=torch.uint8, device=device)
    return GatherBuffers(send, recv, outs, tokens, chunk, hq, d, out_dtype, world)


def all_gather_bytes(send: torch.Tensor, recv: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Rank-major all-gather of equal-size byte buffers: one NCCL all-gather over NVLink
    on GPUs, gloo's list all-gather on the CPU."""
    import torch.distributed as dist

    if world == 1:
        recv.copy_(send)
        return recv
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(recv, send, group=group)
        return recv
    # gloo (CPU tests, or a plumbing check of the TP path on a 1-GPU box): via host memory
    parts = [torch.empty_like(send, device="cpu") for _ in range(world)]
    dist.all_gather(parts, send.cpu(), group=group)
    recv.view(world, -1).copy_(torch.stack(parts))
    return recv


def assemble_layer(gb: GatherBuffers) -> Tuple[torch.Tensor, torch.Tensor]:
    """The rank-major receive buffer -> the layer output O [tokens][Hq][d] and LSE
    [tokens][Hq] (rank t's heads are q heads [t*Hq/T, (t+1)*Hq/T)); rows [0, chunk)
    are the prefill chunk, then one row per decode."""
    w, n, hq, d = gb.world, gb.tokens, gb.hq_rank, gb.head_dim
    per = gb.recv.view(w, -1)
    esz = torch.empty((), dtype=gb.out_dtype).element_size()
    o_bytes = n * hq * d * esz
    o_pad = (o_bytes + 15) // 16 * 16
    o = per[:, :o_bytes].contiguous().view(gb.out_dtype).view(w, n, hq, d)
    lse = per[:, o_pad:].contiguous().view(torch.float32).view(w, n, hq)
    return (o.permute(1, 0, 2, 3).reshape(n, w * hq, d), lse.permute(1, 0, 2).reshape(n, w * hq))


def assemble(gathered: torch.Tensor, world: int, tokens: int, hq_rank: int, d: int) -> torch.Tensor:
    """[world * tokens * hq_rank * d] (rank-major all-gather buffer) -> [tokens][world*hq_rank][d]."""
    return gathered.view(world, tokens, hq_rank, d).permute(1, 0, 2, 3).reshape(tokens, world * hq_rank, d)


def gather_outputs(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gathers each rank's flattened [tokens][Hq/T][d] output into a rank-major
    buffer (one NCCL all-gather over NVLink on GPUs; gloo for CPU tests)."""
    import torch.distributed as dist

    if world == 1:
        return local.reshape(-1)
    flat = local.reshape(-1).contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
        dist.all_gather_into_tensor(out, flat, group=group)
        return out
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat, group=group)
    return torch.cat(parts)


def layer_error(o: torch.Tensor, lse: torch.Tensor, o_ref: torch.Tensor, lse_ref: torch.Tensor,
                group: int) -> Tuple[float, float]:
    """Worst per-KV-head-block error of an assembled layer against a reference layer:
    max |O - O_ref| / max |O_ref| over each (token, KV head) block of `group` q heads
    (the north-star tolerance form), and max |LSE - LSE_ref|."""
    n, hq, d = o_ref.shape
    a = o.float().view(n, hq // group, group * d)
    r = o_ref.float().view(n, hq // group, group * d)
    scale = r.abs().amax(dim=2).clamp_min(1e-30)
    eo = float(((a - r).abs().amax(dim=2) / scale).max())
    fin = torch.isfinite(lse_ref)
    el = float((lse.float() - lse_ref.float())[fin].abs().max()) if bool(fin.any()) else 0.0
    return eo, el


def oproj(o: torch.Tensor, w: torch.Tensor, y_parts, rows_per_rank: int = 0, accumulate: bool = False,
          stream=None) -> None:
    """pod_oproj_run: Y (+)= O W on the GPU (the o_proj consumer).

    o: [tokens][K] bf16 (this rank's heads), w: [K][N] bf16 (their W_o rows).  y_parts:
    one fp32 [rows_per_rank][N] tensor -- or raw device address, e.g. a peer-mapped
    symmetric-memory buffer -- per rank.  accumulate=True reduces every output tile into
    the row owner's Y (the reduce-scatter half of row-parallel TP; Y zeroed beforehand);
    False stores (one rank)."""
    import ctypes as C

    from ._abi import lib
    from .pod import _check

    if o.dtype != torch.bfloat16 or w.dtype != torch.bfloat16 or not o.is_contiguous() or not w.is_contiguous():
        raise ValueError("oproj: o and w must be contiguous bf16")
    tokens, k = o.shape
    if w.shape[0] != k:
        raise ValueError("oproj: o is [tokens][K], w is [K][N]")
    n = w.shape[1]
    ptrs = [p if isinstance(p, int) else p.data_ptr() for p in y_parts]
    for p in y_parts:
        if isinstance(p, torch.Tensor) and (p.dtype != torch.float32 or not p.is_contiguous()):
            raise ValueError("oproj: y parts must be contiguous fp32")
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    st = stream or torch.cuda.current_stream(o.device)
    with torch.cuda.device(o.device):
        _check(lib().pod_oproj_run(C.c_void_p(o.data_ptr()), C.c_void_p(w.data_ptr()), tokens, k, n, arr, len(ptrs),
                                   rows_per_rank or tokens, 1 if accumulate else 0, C.c_void_p(st.cuda_stream)),
               "pod_oproj_run")
