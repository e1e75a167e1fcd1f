"""Full-size GPU parity at every BASELINE config.

Each test runs one BASELINE configuration at its real size through the kernel AUTO
picks (and, where named, through every POD kernel), then checks:

* EVERY (row, q head) of the prefill chunk and EVERY (request, q head) of the decode
  batch against a float64 dense softmax(QK^T / scale) V of the same bf16 inputs,
  computed on the device by plain PyTorch (the checker, not the product path; the
  paged cache is gathered by torch indexing).  This is attention.hpp:148-222 (causal
  prefill, row r sees keys [0, offset + r]) and :240-333 (decode over all ctx keys,
  natural-log LSE) evaluated densely.
* a sample of >= 64 prefill rows and >= 16 decode requests against the pinned CPU
  oracle (tests/common.py -> oracle/, bitwise equal to the compiled reference).

Tolerance (north star): max |O_gpu - O_ref| <= 2e-3 * max |O_ref| per KV-head block
(prefill: all rows x the group's q heads; decode: one request x the group's q heads);
|LSE_gpu - LSE_ref| <= 2e-3 (absolute, natural log).
"""
import math

import pytest
import torch

import paper_2410_18038_b200 as pkg
from paper_2410_18038_b200._abi import POD_POLICY_AUTO, POD_POLICY_COMPLEMENT, POD_POLICY_WARPSPEC
from paper_2410_18038_b200.workload import build_workload, make_batch
from tests.common import LSE_TOL, O_TOL, compare_decode, compare_prefill

pytestmark = pytest.mark.gpu

SCALE = math.sqrt(128)

# name: (Hq, Hkv, chunk, offset, decode batch, decode ctx)   -- SURVEY.md 8 "Configs"
CONFIGS = {
    "c1": (32, 8, 512, 1536, 8, 2048),
    "c2_b8": (32, 8, 1024, 15360, 8, 16384),
    "c2_b16": (32, 8, 1024, 15360, 16, 16384),
    "c2_b32": (32, 8, 1024, 15360, 32, 16384),
    "c2_b64": (32, 8, 1024, 15360, 64, 16384),
    "c3_tp2_rank": (16, 4, 1024, 15360, 64, 16384),
    "c3_tp4_rank": (8, 2, 1024, 15360, 64, 16384),
    "c3_tp8_rank": (4, 1, 1024, 15360, 64, 16384),
    "c4": (32, 32, 2048, 2048, 128, 4096),
}


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _batch(name):
    hq, hkv, chunk, off, nb, ctx = CONFIGS[name]
    return make_batch(pkg.ModelShape(hq, hkv, 128, SCALE), chunk=chunk, offset=off, decode_ctx=[ctx] * nb)


def _gather(wl, req):
    """K, V of request `req` as [ctx][Hkv][d] float64, through the block table (torch indexing)."""
    ctx = wl.kv_lens[req]
    a, b = int(wl.page_indptr[req]), int(wl.page_indptr[req + 1])
    pages = wl.page_indices[a:b].long()
    hkv, d = wl.k_pool.shape[1], wl.k_pool.shape[3]
    k = wl.k_pool[pages].permute(0, 2, 1, 3).reshape(-1, hkv, d)[:ctx]
    v = wl.v_pool[pages].permute(0, 2, 1, 3).reshape(-1, hkv, d)[:ctx]
    return k.double(), v.double()


def _dense_head(q, k, v, scale, limit):
    """q [m][G][d], k/v [n][d] float64; row r sees keys j <= limit[r].  -> O [m][G][d], LSE [m][G]."""
    s = torch.einsum("rgd,jd->grj", q, k) / scale
    j = torch.arange(k.shape[0], device=q.device)
    s = s.masked_fill(j[None, None, :] > limit[None, :, None], float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    o = torch.einsum("grj,jd->rgd", torch.softmax(s, dim=-1), v)
    return o, lse.transpose(0, 1)


def _check_dense(wl, out):
    """Every row / request / q head against the float64 dense reference; returns the worst errors."""
    b = wl.batch
    G, hkv = b.shape.group_size(), b.shape.num_kv_heads
    worst = {"prefill_o": 0.0, "prefill_lse": 0.0, "decode_o": 0.0, "decode_lse": 0.0}
    req0 = 0
    if b.prefill is not None:
        k, v = _gather(wl, 0)
        m, off = b.prefill.chunk_size, b.prefill.position_offset
        lim = off + torch.arange(m, device=k.device)
        qp = wl.q_prefill.double().view(m, hkv, G, -1)
        op = out.o_prefill.double().view(m, hkv, G, -1)
        lp = out.lse_prefill.double().view(m, hkv, G)
        for h in range(hkv):
            o_ref, l_ref = _dense_head(qp[:, h], k[:, h], v[:, h], b.shape.scale, lim)
            e = ((op[:, h] - o_ref).abs().max() / o_ref.abs().max()).item()
            el = (lp[:, h] - l_ref).abs().max().item()
            worst["prefill_o"] = max(worst["prefill_o"], e)
            worst["prefill_lse"] = max(worst["prefill_lse"], el)
        req0 = 1
    for i in range(len(b.decodes)):
        k, v = _gather(wl, req0 + i)
        lim = torch.tensor([k.shape[0] - 1], device=k.device)
        qd = wl.q_decode[i].double().view(1, hkv, G, -1)
        od = out.o_decode[i].double().view(hkv, G, -1)
        ld = out.lse_decode[i].double().view(hkv, G)
        for h in range(hkv):
            o_ref, l_ref = _dense_head(qd[:, h], k[:, h], v[:, h], b.shape.scale, lim)
            e = ((od[h] - o_ref[0]).abs().max() / o_ref.abs().max()).item()
            worst["decode_o"] = max(worst["decode_o"], e)
            worst["decode_lse"] = max(worst["decode_lse"], (ld[h] - l_ref[0]).abs().max().item())
    assert torch.isfinite(out.o_prefill if b.prefill is not None else out.o_decode).all()
    assert worst["prefill_o"] <= O_TOL and worst["decode_o"] <= O_TOL, worst
    assert worst["prefill_lse"] <= LSE_TOL and worst["decode_lse"] <= LSE_TOL, worst
    return worst


def _check_oracle_sample(wl, out):
    """>= 64 prefill rows (both ends and the middle of the chunk, 2 KV heads) and >= 16
    decode requests (2 KV heads) against the pinned CPU oracle."""
    b = wl.batch
    hkv = b.shape.num_kv_heads
    heads = sorted({0, hkv - 1})
    if b.prefill is not None:
        m = b.prefill.chunk_size
        o_p, l_p = out.o_prefill.cpu().numpy(), out.lse_prefill.cpu().numpy()
        for r0 in (0, m // 2 - 16, m - 32):
            eo, el = compare_prefill(wl, o_p, l_p, kv_heads=heads, row_range=(r0, r0 + 32))
            assert eo <= O_TOL and el <= LSE_TOL, ("oracle prefill", r0, eo, el)
    nb = len(b.decodes)
    reqs = sorted(set(range(0, nb, max(1, nb // 16))) | {nb - 1})
    eo, el = compare_decode(wl, out.o_decode.cpu().numpy(), out.lse_decode.cpu().numpy(), requests=reqs,
                            kv_heads=heads)
    assert eo <= O_TOL and el <= LSE_TOL, ("oracle decode", eo, el)


def _run(wl, batch, policy=POD_POLICY_AUTO, keys=0, s_buffers=0):
    from paper_2410_18038_b200.hybrid import PodAttention

    opts = pkg.PlanOptions(policy=policy, prefill_tile_keys=keys, prefill_s_buffers=s_buffers)
    op = PodAttention(batch, options=opts)
    out = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)
    torch.cuda.synchronize()
    return op, out


@pytest.mark.parametrize("name", list(CONFIGS))
def test_baseline_config_full_size_auto(name):
    """The kernel AUTO picks, every row / request / head against the dense reference,
    plus the oracle sample."""
    _need_gpu()
    batch = _batch(name)
    wl = build_workload(batch, device="cuda")
    op, out = _run(wl, batch)
    assert op.info.policy in (POD_POLICY_WARPSPEC, POD_POLICY_COMPLEMENT)
    worst = _check_dense(wl, out)
    _check_oracle_sample(wl, out)
    print(f"{name}: policy {op.info.policy} keys {op.info.prefill_tile_keys} worst {worst}")


@pytest.mark.parametrize("name", ["c2_b16", "c2_b64"])
def test_baseline_config_full_size_peaky(name):
    """Peaky queries (Q x 8: sharp softmax, online-softmax rescales on the early tiles)
    at the 64-key (C2 B=16) and 32-key (C2 B=64) pair-engine points."""
    _need_gpu()
    batch = _batch(name)
    wl = build_workload(batch, device="cuda", q_scale=8.0)
    op, out = _run(wl, batch)
    assert op.info.prefill_tile_keys == (64 if name == "c2_b16" else 32)
    _check_dense(wl, out)


@pytest.mark.parametrize("name", ["c2_b16", "c4"])
@pytest.mark.parametrize("kernel", [(POD_POLICY_COMPLEMENT, 0), (POD_POLICY_WARPSPEC, 32), (POD_POLICY_WARPSPEC, 64, 1),
                                    (POD_POLICY_WARPSPEC, 64, 2)])
def test_baseline_config_full_size_every_kernel(name, kernel):
    """Both POD kernels (and every pair engine) forced at C2 B=16 and C4."""
    _need_gpu()
    batch = _batch(name)
    wl = build_workload(batch, device="cuda")
    op, out = _run(wl, batch, *kernel)
    assert op.info.policy == kernel[0]
    _check_dense(wl, out)


@pytest.mark.parametrize("chunk,ctx,nb", [(512, 65536, 8), (4096, 16384, 8)])
def test_c5_extremes_full_size(chunk, ctx, nb):
    """C5 sweep corners (BASELINE configs[4]): a 64K context and a 4K chunk, through the
    kernel AUTO picks, every row / request / head against the dense reference."""
    _need_gpu()
    batch = make_batch(pkg.ModelShape(32, 8, 128, SCALE), chunk=chunk, offset=ctx - chunk, decode_ctx=[ctx] * nb)
    wl = build_workload(batch, device="cuda")
    op, out = _run(wl, batch)
    worst = _check_dense(wl, out)
    print(f"{chunk}@{ctx}+{nb}: policy {op.info.policy} keys {op.info.prefill_tile_keys} worst {worst}")
