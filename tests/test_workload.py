"""Synthetic inputs and the paged-KV integer mapping (bit-exact).

Logical token t of request i lives in page page_indices[page_indptr[i] + t/16]
at slot t%16; gathering the bf16 pool through the block table must reproduce
the reference's contiguous KVCacheT layout (attention.hpp:36-38) exactly."""
import math

import numpy as np
import torch

from oracle import pyoracle as O
from paper_2410_18038_b200 import ModelShape
from paper_2410_18038_b200.workload import Rng, build_workload, make_batch, rng_doubles, rng_permutation, rng_values


def test_rng_vectorised_equals_sequential():
    r = Rng(43)
    seq = [r.next_double() for _ in range(100)]
    assert np.array_equal(np.array(seq), rng_doubles(43, 0, 100).numpy())
    # a slice can be regenerated anywhere in the stream
    assert np.array_equal(rng_doubles(43, 37, 20).numpy(), np.array(seq[37:57]))


def test_rng_values_bf16_rounding():
    x = rng_values(42, 0, 1000)
    ref = (rng_doubles(42, 0, 1000) * 2 - 1).to(torch.float32).to(torch.bfloat16)
    assert torch.equal(x, ref)


def test_page_permutation_is_a_permutation():
    p = rng_permutation(44, 1000)
    assert sorted(p) == list(range(1000)) and p != list(range(1000))


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).numpy().view(np.uint16)


def test_paged_gather_is_bit_exact_hnd_and_nhd():
    shape = ModelShape(8, 2, 128, math.sqrt(128))
    batch = make_batch(shape, chunk=20, offset=37, decode_ctx=[1, 15, 16, 17, 100])
    wl = build_workload(batch, pad_value=7.0)
    ip, ix = wl.page_indptr.numpy(), wl.page_indices.numpy()
    pool_hnd = _bits(wl.k_pool)
    pool_nhd = np.ascontiguousarray(pool_hnd.transpose(0, 2, 1, 3))
    for req, ctx in enumerate(wl.kv_lens):
        ref = wl.request_cache(req, "k").numpy()
        assert np.array_equal(O.gather_pages(pool_hnd, 0, ip, ix, req, ctx), ref)
        assert np.array_equal(O.gather_pages(pool_nhd, 1, ip, ix, req, ctx), ref)
        refv = wl.request_cache(req, "v").numpy()
        assert np.array_equal(O.gather_pages(_bits(wl.v_pool), 0, ip, ix, req, ctx), refv)
        # one-head regeneration equals the full cache's slice
        for h in range(shape.num_kv_heads):
            assert np.array_equal(wl.request_cache(req, "k", head=h).numpy(), ref[:, h, :])


def test_padding_and_block_table_layout():
    shape = ModelShape(4, 1, 128, 1.0)
    wl = build_workload(make_batch(shape, decode_ctx=[17]), pad_value=3.0)
    ip, ix = wl.page_indptr.tolist(), wl.page_indices.tolist()
    assert ip == [0, 2]
    last = wl.k_pool[ix[1]]  # [Hkv][16][d]; slots 1..15 of the 2nd page are padding
    assert torch.all(last[:, 1:, :].float() == 3.0)
    assert len(set(ix)) == len(ix)


def test_gather_out_of_range_page_is_rejected():
    pool = np.zeros((2, 1, 16, 128), np.uint16)
    try:
        O.gather_pages(pool, 0, np.array([0, 1], np.int32), np.array([5], np.int32), 0, 4)
    except O.OracleError as e:
        assert e.status == 4
    else:
        raise AssertionError("expected out_of_range")


def test_kv_append_oracle_round_trip_hnd_and_nhd():
    """Oracle KV append (test infrastructure): zero the new tokens' slots, scatter the
    rows back through the block table -> the pool is bit-identical again (both layouts),
    and the rows are what gather_pages reads at those positions."""
    from tests.common import new_token_rows, token_slots

    shape = ModelShape(8, 2, 128, math.sqrt(128))
    batch = make_batch(shape, chunk=20, offset=37, decode_ctx=[1, 15, 16, 17, 100])
    wl = build_workload(batch, pad_value=7.0)
    ip, ix = wl.page_indptr.numpy(), wl.page_indices.numpy()
    kp, vp, kd, vd = new_token_rows(wl)
    slots = token_slots(wl)
    for layout in (0, 1):
        full = _bits(wl.k_pool)
        if layout == 1:
            full = np.ascontiguousarray(full.transpose(0, 2, 1, 3))
        pool = full.copy()
        for page, slot in slots:
            if layout == 0:
                pool[page, :, slot, :] = 0
            else:
                pool[page, slot, :, :] = 0
        assert not np.array_equal(pool, full)
        O.append_kv(pool, layout, ip, ix, 0, batch.prefill.position_offset, kp)
        for i, d in enumerate(batch.decodes):
            O.append_kv(pool, layout, ip, ix, 1 + i, d.context_len - 1, kd[i:i + 1])
        assert np.array_equal(pool, full)
    assert kp.shape == (20, 2, 128) and kd.shape == (5, 2, 128) and vp.shape == kp.shape and vd.shape == kd.shape
