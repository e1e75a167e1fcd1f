"""KV-head-group tensor parallelism, world_size 2 over gloo (CPU).

Each rank computes attention for its own KV heads (the CPU oracle stands in for
the GPU kernel here), the outputs are all-gathered and assembled; the result
must equal the unsharded layer exactly (attention is independent per KV head,
SURVEY.md 8(e))."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_18038_b200 import ModelShape
from paper_2410_18038_b200.tp import assemble, gather_outputs, shard_heads
from paper_2410_18038_b200.workload import build_workload, make_batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _layer(shape, kv_heads):
    from tests.common import oracle_decode, oracle_prefill

    batch = make_batch(shape, chunk=24, offset=40, decode_ctx=[33, 70])
    wl = build_workload(batch)
    G = shape.group_size()
    pf = oracle_prefill(wl, kv_heads=kv_heads)
    dc = oracle_decode(wl, kv_heads=kv_heads)
    o_p = np.concatenate([pf[h][0] for h in kv_heads], axis=1)            # [chunk][G*len][d]
    o_d = np.stack([np.concatenate([dc[(r, h)][0] for h in kv_heads], axis=0) for r in range(2)])
    return np.concatenate([o_p, o_d], axis=0)                               # [tokens][Hq_rank][d]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = ModelShape(8, 4, 128, math.sqrt(128))
    sh = shard_heads(shape, rank, world)
    local = torch.from_numpy(_layer(shape, list(range(sh.kv_head_begin, sh.kv_head_end))))
    full = gather_outputs(local, world)
    if rank == 0:
        tokens = local.shape[0]
        q.put(assemble(full, world, tokens, sh.shape.num_q_heads, 128).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_heads():
    s = ModelShape(32, 8, 128, 1.0)
    shards = [shard_heads(s, r, 4) for r in range(4)]
    assert [(x.kv_head_begin, x.kv_head_end, x.q_head_begin, x.q_head_end) for x in shards] == \
        [(0, 2, 0, 8), (2, 4, 8, 16), (4, 6, 16, 24), (6, 8, 24, 32)]
    assert all(x.shape.num_q_heads == 8 and x.shape.num_kv_heads == 2 for x in shards)
    with pytest.raises(ValueError):
        shard_heads(s, 0, 3)


def test_tp2_gloo_all_gather_equals_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    shape = ModelShape(8, 4, 128, math.sqrt(128))
    ref = _layer(shape, list(range(4)))
    assert np.array_equal(got, ref)
