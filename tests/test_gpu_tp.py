"""The KV-head-group TP path end to end on ONE GPU.

For T in {2, 4, 8}, every "rank" slices the same seeded layer (`tp.shard_workload`),
plans its own shape, runs the real fused kernel straight into its all-gather send
buffer (`tp.gather_buffers`); the T send buffers are laid rank-major into one
receive buffer (what the NCCL all-gather produces) and assembled
(`tp.assemble_layer`).  The assembled layer must match a TP1 fused run of the same
layer and a float64 dense reference within the north-star bound -- the same
functions bench.py runs under torchrun, minus only the collective itself.
"""
import math

import pytest
import torch

import paper_2410_18038_b200 as pkg
from paper_2410_18038_b200.hybrid import PodAttention
from paper_2410_18038_b200.tp import assemble_layer, gather_buffers, layer_error, shard_heads, shard_workload
from paper_2410_18038_b200.workload import build_workload, make_batch
from tests.common import dense_layer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_tp_sharded_layer_on_one_gpu(world, out_dtype):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    shape = pkg.ModelShape(32, 8, 128, math.sqrt(128))
    batch = make_batch(shape, chunk=256, offset=1792, decode_ctx=[2048, 1500, 777, 2048, 16, 3000])
    full = build_workload(batch, device="cuda")
    odt = 0 if out_dtype == torch.float32 else 1
    gbs = []
    for r in range(world):
        wl = shard_workload(full, shard_heads(shape, r, world))
        gb = gather_buffers(wl.batch, world, out_dtype, "cuda")
        PodAttention(wl.batch, options=pkg.PlanOptions(out_dtype=odt)).run(
            wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, out=gb.outputs)
        gbs.append(gb)
    torch.cuda.synchronize()
    g0 = gbs[0]
    g0.recv.view(world, -1).copy_(torch.stack([g.send for g in gbs]))  # the all-gather's result
    o, lse = assemble_layer(g0)
    ro = PodAttention(batch, options=pkg.PlanOptions(out_dtype=odt)).run(
        full.q_prefill, full.q_decode, full.k_pool, full.v_pool, full.page_indptr, full.page_indices)
    o1 = torch.cat([ro.o_prefill, ro.o_decode])
    l1 = torch.cat([ro.lse_prefill, ro.lse_decode])
    o_ref, lse_ref = dense_layer(full)
    tol = 2e-3 if out_dtype == torch.float32 else 8e-3  # bf16 outputs: + 2^-8 rounding of O
    eo, el = layer_error(o, lse, o1, l1, shape.group_size())
    assert eo <= tol and el <= 2e-3, ("vs tp1", eo, el)
    eo, el = layer_error(o, lse, o_ref, lse_ref, shape.group_size())
    assert eo <= tol and el <= 2e-3, ("vs dense", eo, el)
