"""Pins the CPU oracle (oracle/pod_oracle.c, test infrastructure) to the reference.

* against tests/golden/attention_golden.npz, produced by the reference's own
  headers (oracle/_ref) on the cases of proj/tests/test_attention.cpp;
* against the reference tests' own assertions (ported case by case);
* against oracle/_ref directly on random cases, where that library is present.
"""
import itertools
import math

import numpy as np
import pytest

import cases
from oracle import pyoracle as O
from paper_2410_18038_b200.workload import Rng, rng_doubles

GOLD = np.load(cases.__file__.replace("cases.py", "attention_golden.npz"))


# ------------------------------------------------------------ golden pins --
def test_rng_matches_reference_draws():
    # rng.hpp:11-47, first 64 draws of every seed the tests use
    for seed in (42, 43, 44, 2024, 4242):
        assert np.array_equal(rng_doubles(seed, 0, 64).numpy(), GOLD[f"rng/{seed}"])
        r = Rng(seed)
        assert [r.next_double() for _ in range(8)] == list(GOLD[f"rng/{seed}"][:8])


def test_naive_seed42_golden():
    q, k, v = cases.naive42()
    assert np.array_equal(O.naive_attention(q, k, v, 2.0), GOLD["naive42/out"])
    assert np.array_equal(O.naive_attention(q, k, v, 2.0, causal_offset=5), GOLD["naive42/out_causal5"])


@pytest.mark.parametrize("gen", [cases.prefill_named, cases.prefill_random2024])
def test_tiled_prefill_golden(gen):
    n = 0
    for name, (chunk, ctx, off, hq, hkv, d), tiles, (q, k, v) in gen():
        for tq, tkv in tiles:
            got = O.tiled_prefill(q, k, v, off, hq, hkv, math.sqrt(d), tq, tkv)
            ref = GOLD[f"{name}/out_{tq}_{tkv}"]
            assert np.array_equal(got, ref), (name, np.abs(got - ref).max())
            n += 1
        if f"{name}/lse" in GOLD.files:
            lse = O.prefill_lse(q, k, off, hq, hkv, math.sqrt(d))
            assert np.allclose(lse, GOLD[f"{name}/lse"], rtol=0, atol=1e-13), name
    assert n >= 5


@pytest.mark.parametrize("gen", [cases.decode_named, cases.decode_random4242])
def test_decode_splitk_and_merge_golden(gen):
    for name, (ctx, hq, hkv, d), splits, (q, k, v) in gen():
        for s in splits:
            o, lse, rg = O.decode_splitk(q, k, v, hq, hkv, math.sqrt(d), s)
            assert np.array_equal(lse, GOLD[f"{name}/lse_{s}"]), (name, s)
            assert np.array_equal(rg, GOLD[f"{name}/rg_{s}"]), (name, s)
            if f"{name}/o_{s}" in GOLD.files:
                assert np.array_equal(o, GOLD[f"{name}/o_{s}"]), (name, s)
            assert np.array_equal(O.merge_partials(o, lse, rg), GOLD[f"{name}/merged_{s}"]), (name, s)


# -------------------------------------- reference test assertions, ported --
def test_naive_one_key_identity():  # test_attention.cpp:109-117
    o = O.naive_attention(np.array([[3.0, 4.0]]), np.array([[1.0, 0.0]]), np.array([[7.0, 9.0]]), 1.0)
    assert o[0, 0] == 7.0 and o[0, 1] == 9.0


def test_naive_identical_keys_average_v():  # :119-129
    q = np.array([[0.3, -1.2]])
    k = np.array([[0.5, -0.25], [0.5, -0.25]])
    v = np.array([[0.0, 0.0], [2.0, 4.0]])
    o = O.naive_attention(q, k, v, 1.0)
    assert abs(o[0, 0] - 1.0) < 1e-12 and abs(o[0, 1] - 2.0) < 1e-12


def test_naive_rows_normalized():  # :144-157
    r = Rng(7)
    q = r.fill_uniform(96).numpy().reshape(12, 8)
    k = r.fill_uniform(160).numpy().reshape(20, 8)
    v = np.ones((20, 8))
    for causal in (None, 5):
        o = O.naive_attention(q, k, v, 3.0, causal_offset=causal)
        assert np.abs(o - 1.0).max() < 1e-12


def test_naive_error_paths():  # :159-166
    with pytest.raises(O.OracleError) as e:
        O.naive_attention(np.zeros((2, 3)), np.zeros((4, 3)), np.zeros((4, 3)), 1.0, causal_offset=-1)
    assert e.value.status == 3  # domain_error: fully masked row
    with pytest.raises(O.OracleError) as e:
        O.naive_attention(np.zeros((0, 3)), np.zeros((4, 3)), np.zeros((4, 3)), 1.0)
    assert e.value.status == 1


def test_gqa_mapping():  # :168-190
    assert O.gqa_kv_head(9, 32, 4) == 1
    for h in range(8):
        assert O.gqa_kv_head(h, 8, 8) == h
    hits = [0] * 8
    prev = 0
    for h in range(32):
        kv = O.gqa_kv_head(h, 32, 8)
        assert kv == h // 4 and kv >= prev
        prev = kv
        hits[kv] += 1
    assert hits == [4] * 8
    with pytest.raises(O.OracleError) as e:
        O.gqa_kv_head(32, 32, 8)
    assert e.value.status == 4


def test_tiled_causality_bitwise():  # :229-244
    _, _, _, (q, k, v) = next((c[0], c[1], c[2], c[3]) for c in cases.prefill_named() if c[0] == "p99")
    off = 20
    before = O.tiled_prefill(q, k, v, off, 2, 1, math.sqrt(8), 3, 8)
    k2, v2 = k.copy(), v.copy()
    k2[off + 3:] += 17.0
    v2[off + 3:] -= 5.0
    after = O.tiled_prefill(q, k2, v2, off, 2, 1, math.sqrt(8), 3, 8)
    assert np.array_equal(before[:3], after[:3])


def test_tiled_cache_too_short():  # :246-250
    r = Rng(1)
    q = r.fill_uniform(8 * 2 * 4).numpy().reshape(8, 2, 4)
    k = r.fill_uniform(10 * 4).numpy().reshape(10, 1, 4)
    with pytest.raises(O.OracleError) as e:
        O.tiled_prefill(q, k, k, 4, 2, 1, 2.0, 4, 4)
    assert e.value.status == 2


def test_gqa_consistency():  # :252-270
    _, _, _, (q, k, v) = next(c for c in cases.prefill_named() if c[0] == "p31")
    grouped = O.tiled_prefill(q, k, v, 16, 8, 2, math.sqrt(8), 4, 8)
    wide_k = np.repeat(k, 4, axis=1)
    wide_v = np.repeat(v, 4, axis=1)
    flat = O.tiled_prefill(q, wide_k, wide_v, 16, 8, 8, math.sqrt(8), 4, 8)
    assert np.abs(grouped - flat).max() <= 1e-12 * np.abs(flat).max()


def test_split_partition_and_clamp():  # :315-324, :350-357
    assert O.split_ranges(12, 4) == [(0, 3), (3, 6), (6, 9), (9, 12)]
    r = Rng(6)
    q = r.fill_uniform(8).numpy().reshape(2, 4)
    k = r.fill_uniform(20).numpy().reshape(5, 1, 4)
    o, lse, rg = O.decode_splitk(q, k, k, 2, 1, 2.0, 64)
    assert len(rg) == 5
    with pytest.raises(O.OracleError) as e:
        O.decode_splitk(q, np.zeros((0, 1, 4)), np.zeros((0, 1, 4)), 2, 1, 2.0, 2)
    assert e.value.status == 3


def test_merge_identity_and_permutation_bitwise():  # :359-365, :381-394
    _, _, _, (q, k, v) = next(c for c in cases.decode_named() if c[0] == "d21")
    o, lse, rg = O.decode_splitk(q, k, v, 4, 2, math.sqrt(8), 4)
    base = O.merge_partials(o, lse, rg)
    for perm in itertools.permutations(range(4)):
        m = O.merge_partials(o[list(perm)], lse[list(perm)], rg[list(perm)])
        assert np.array_equal(m, base)
    o1, l1, r1 = O.decode_splitk(q, k, v, 4, 2, math.sqrt(8), 1)
    assert np.array_equal(O.merge_partials(o1, l1, r1), o1[0])


def test_merge_overlap_rejected():  # :396-403
    _, _, _, (q, k, v) = next(c for c in cases.decode_named() if c[0] == "d3")
    o, lse, rg = O.decode_splitk(q, k, v, 2, 1, 2.0, 2)
    rg = rg.copy()
    rg[1, 0] = rg[0, 1] - 1
    with pytest.raises(O.OracleError) as e:
        O.merge_partials(o, lse, rg)
    assert e.value.status == 2
    with pytest.raises(O.OracleError):
        O.merge_partials(np.zeros((0, 2, 4)), np.zeros((0, 2)), np.zeros((0, 2), np.int64))


def test_split_invariance():  # :326-334
    _, _, _, (q, k, v) = next(c for c in cases.decode_named() if c[0] == "d77")
    base = O.merge_partials(*O.decode_splitk(q, k, v, 4, 2, 4.0, 1))
    for s in (2, 4, 8):
        m = O.merge_partials(*O.decode_splitk(q, k, v, 4, 2, 4.0, s))
        assert np.abs(m - base).max() <= 1e-10 * np.abs(base).max()


# ------------------------------------------------ port == compiled reference --
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_port_equals_reference_random():
    rs = np.random.default_rng(3)
    for it in range(12):
        d = int(rs.choice([4, 8, 16, 64]))
        hkv = int(rs.integers(1, 3))
        hq = hkv * int(rs.integers(1, 5))
        chunk = int(rs.integers(1, 40))
        off = int(rs.integers(0, 200))
        ctx = off + chunk + int(rs.integers(0, 30))
        q = rs.uniform(-1, 1, (chunk, hq, d))
        k = rs.uniform(-1, 1, (ctx, hkv, d))
        v = rs.uniform(-1, 1, (ctx, hkv, d))
        tq, tkv = int(rs.choice([1, 8, 64])), int(rs.choice([1, 7, 64, 128]))
        a = O.tiled_prefill(q, k, v, off, hq, hkv, math.sqrt(d), tq, tkv, which="port")
        b = O.tiled_prefill(q, k, v, off, hq, hkv, math.sqrt(d), tq, tkv, which="ref")
        assert np.array_equal(a, b)
        s = int(rs.integers(1, 9))
        pa = O.decode_splitk(q[0], k, v, hq, hkv, math.sqrt(d), s, which="port")
        pb = O.decode_splitk(q[0], k, v, hq, hkv, math.sqrt(d), s, which="ref")
        for x, y in zip(pa, pb):
            assert np.array_equal(x, y)
        assert np.array_equal(O.merge_partials(*pa, which="port"), O.merge_partials(*pb, which="ref"))
