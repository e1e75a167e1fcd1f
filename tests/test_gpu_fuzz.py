"""Random hybrid batches on the GPU, every kernel, checked row by row.

48 seeded cases: GQA group 1/2/4/8, ragged decode contexts (1 .. 3000 keys, page edges
included), chunks of 1 .. 300 rows at random offsets (0 included), prefill-only and
decode-only batches, uniform and peaky (Q x 8) queries, and every kernel the plan can
pick (AUTO, the two-CTA kernel, the warp-specialised kernel with its 32-key and 64-key
pair engines).  Every (row, q head) and (request, q head) is compared with a float64
dense softmax(QK^T / scale) V of the same bf16 inputs gathered through the block table
(tests/common.py::dense_layer; semantics attention.hpp:148-222, :240-333), at the
north-star bound: max |O - O_ref| <= 2e-3 * max |O_ref| per (token, KV head) block,
|LSE - LSE_ref| <= 2e-3.
"""
import math
import random

import pytest
import torch

import paper_2410_18038_b200 as pkg
from paper_2410_18038_b200._abi import POD_POLICY_AUTO, POD_POLICY_COMPLEMENT, POD_POLICY_WARPSPEC
from paper_2410_18038_b200.tp import layer_error
from paper_2410_18038_b200.workload import build_workload, make_batch
from tests.common import LSE_TOL, O_TOL, dense_layer

pytestmark = pytest.mark.gpu

KERNELS = [
    ("auto", dict(policy=POD_POLICY_AUTO)),
    ("complement", dict(policy=POD_POLICY_COMPLEMENT)),
    ("ws32", dict(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=32)),
    ("ws64", dict(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=64, prefill_s_buffers=1)),
    ("ws64db", dict(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=64, prefill_s_buffers=2)),
]


def _case(i):
    rng = random.Random(1000 + i)
    hkv = rng.choice([1, 2, 4, 8])
    g = rng.choice([1, 2, 4, 8])
    d = random.Random(5000 + i).choice([128, 128, 128, 64, 32])  # head dims < 128 run zero-padded
    shape = pkg.ModelShape(hkv * g, hkv, d, math.sqrt(d))
    kind = rng.random()
    chunk = 0 if kind < 0.15 else rng.randint(1, 300)
    offset = 0 if chunk and rng.random() < 0.2 else rng.randint(0, 2000)
    nb = 0 if (0.15 <= kind < 0.25 and chunk) else rng.randint(1, 12)
    ctx = [rng.choice([1, 15, 16, 17]) if rng.random() < 0.3 else rng.randint(1, 3000) for _ in range(nb)]
    q_scale = rng.choice([1.0, 1.0, 8.0])
    name, opts = KERNELS[i % len(KERNELS)]
    return shape, chunk, offset if chunk else 0, ctx, q_scale, name, opts


@pytest.mark.parametrize("i", range(48))
def test_random_hybrid_batch(i):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2410_18038_b200.hybrid import PodAttention

    shape, chunk, offset, ctx, q_scale, name, opts = _case(i)
    batch = make_batch(shape, chunk=chunk, offset=offset, decode_ctx=ctx)
    wl = build_workload(batch, device="cuda", q_scale=q_scale, seed_q=42 + i, seed_kv=43 + i)
    try:
        op = PodAttention(batch, options=pkg.PlanOptions(**opts))
    except pkg.Unsupported:
        pytest.skip(f"{name} does not run this shape")  # e.g. the pair engine with > 256-row q tiles
    out = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)
    torch.cuda.synchronize()
    o = torch.cat([t for t in (out.o_prefill, out.o_decode) if t is not None])
    lse = torch.cat([t for t in (out.lse_prefill, out.lse_decode) if t is not None])
    o_ref, lse_ref = dense_layer(wl)
    eo, el = layer_error(o, lse, o_ref, lse_ref, shape.group_size())
    assert torch.isfinite(o).all()
    assert eo <= O_TOL and el <= LSE_TOL, (name, shape, chunk, offset, ctx, q_scale, eo, el)
