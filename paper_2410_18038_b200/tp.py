"""KV-head-group tensor parallelism for the hybrid-batch layer.

Rank t of T owns KV heads [t*Hkv/T, (t+1)*Hkv/T) and their `group` query heads,
so attention needs no exchange; one all-gather of the per-rank outputs
[tokens][Hq/T][d] assembles the layer output [tokens][Hq][d].
"""
from __future__ import annotations

from dataclasses import dataclass

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
