"""KV-head-group tensor parallelism, world_size 2 over gloo (CPU).

Each rank slices the SAME seeded full-layer workload with bench.py's own helpers
(`tp.shard_workload`), computes its heads' attention (a float64 dense stand-in
for the GPU kernel, which this CPU container cannot run -- the GPU test
`test_gpu_parity.py::test_tp_sharded_layer_on_one_gpu` runs the real kernels
through the same path), writes it into the all-gather send buffer
(`tp.gather_buffers`), all-gathers (`tp.all_gather_bytes`) and assembles
(`tp.assemble_layer`); rank 0's assembled layer must equal the unsharded layer
(attention is independent per KV head)."""
import math
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_18038_b200 import ModelShape
from paper_2410_18038_b200.tp import (all_gather_bytes, assemble_layer, gather_buffers, layer_error, shard_heads,
                                      shard_workload)
from paper_2410_18038_b200.workload import build_workload, make_batch

SHAPE = ModelShape(8, 4, 128, math.sqrt(128))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _full_workload():
    return build_workload(make_batch(SHAPE, chunk=24, offset=40, decode_ctx=[33, 70, 5]))


def _worker(rank, world, port, q, out_dtype):
    from tests.common import dense_layer

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = shard_heads(SHAPE, rank, world)
    wl = shard_workload(_full_workload(), sh)
    gb = gather_buffers(wl.batch, world, out_dtype, "cpu")
    o, lse = dense_layer(wl)           # the rank's heads: [tokens][Hq/T][d], [tokens][Hq/T]
    c = wl.batch.prefill.chunk_size
    gb.outputs.o_prefill.copy_(o[:c])
    gb.outputs.lse_prefill.copy_(lse[:c])
    gb.outputs.o_decode.copy_(o[c:])
    gb.outputs.lse_decode.copy_(lse[c:])
    all_gather_bytes(gb.send, gb.recv, world)
    if rank == 0:
        q.put(tuple(t.clone() for t in assemble_layer(gb)))
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


def test_shard_workload_slices_pools_and_queries():
    wl = _full_workload()
    sh = shard_heads(SHAPE, 1, 2)
    r = shard_workload(wl, sh)
    assert r.batch.shape.num_q_heads == 4 and r.batch.shape.num_kv_heads == 2
    assert torch.equal(r.k_pool, wl.k_pool[:, 2:4]) and torch.equal(r.v_pool, wl.v_pool[:, 2:4])
    assert torch.equal(r.q_prefill, wl.q_prefill[:, 4:8]) and torch.equal(r.q_decode, wl.q_decode[:, 4:8])
    assert r.k_pool.is_contiguous() and r.q_decode.is_contiguous()
    assert torch.equal(r.page_indptr, wl.page_indptr) and torch.equal(r.page_indices, wl.page_indices)


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_tp2_gloo_all_gather_equals_unsharded(out_dtype):
    from tests.common import dense_layer

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, out_dtype)) for r in range(2)]
    for p in procs:
        p.start()
    o, lse = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full = _full_workload()
    # exact: the gathered + assembled bytes are each rank's outputs at their head columns
    parts = [dense_layer(shard_workload(full, shard_heads(SHAPE, r, 2))) for r in range(2)]
    assert torch.equal(o, torch.cat([p[0] for p in parts], dim=1).to(out_dtype))
    assert torch.equal(lse, torch.cat([p[1] for p in parts], dim=1).float())
    # and the assembled layer is the unsharded layer (fp32: within the north-star bound;
    # a bf16 output carries its own 2^-8 rounding, checked exactly above)
    o_ref, lse_ref = dense_layer(full)
    assert o.shape == o_ref.shape and lse.shape == lse_ref.shape
    if out_dtype == torch.float32:
        eo, el = layer_error(o, lse, o_ref, lse_ref, SHAPE.group_size())
        assert eo <= 1e-6 and el <= 1e-6
