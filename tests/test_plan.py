"""Host planner (pod_attn_plan) parity with the reference's work decomposition.

Ports the assertions of proj/tests/test_work_decomp.cpp and the scheduler cases
of proj/tests/test_gpu_sim.cpp:80-114, and compares the task table field by
field against decompose_hybrid() compiled from the reference (oracle/_ref).
"""
import math
import random

import numpy as np
import pytest

import paper_2410_18038_b200 as pkg
from oracle import pyoracle as O
from paper_2410_18038_b200 import (DecodeSpec, GpuSpec, HybridBatchSpec, InvalidArgument, ModelShape, Plan,
                                   PlanOptions, PrefillSpec, TileConfig, decompose_hybrid, limit_prefill_splits,
                                   make_tile_config, select_tile_config)
from paper_2410_18038_b200._abi import POD_TILE_B200, POD_TILE_REFERENCE

YI = ModelShape(32, 4, 128, 11.3137)
LLAMA_TP2 = ModelShape(16, 4, 128, 11.3137)


def decode_batch(n, ctx, shape=YI):
    return HybridBatchSpec(decodes=[DecodeSpec(ctx)] * n, shape=shape)


def ref_cfg(cfg: TileConfig):
    return O.RefTileConfig(cfg.prefill_tile_q, cfg.decode_tile_q, cfg.tile_kv, cfg.warps_per_cta, cfg.ctas_per_sm,
                           cfg.shared_mem_per_cta, int(cfg.virtual_decode), cfg.split_wave_cap)


def ref_gpu(g: GpuSpec):
    return O.RefGpuSpec(g.num_sms, g.compute_rate_per_sm, g.mem_bandwidth_total, g.mem_bandwidth_per_sm,
                        g.mem_interference, g.max_ctas_per_sm, g.shared_mem_per_sm)


# ------------------------------------------------- test_work_decomp.cpp ---
def test_decode_one_cta_per_request_kv_head():  # :35-53
    gpu = GpuSpec.reference_default()
    t54 = decompose_hybrid(decode_batch(54, 16384), gpu, TileConfig()).decode_tasks
    t55 = decompose_hybrid(decode_batch(55, 16384), gpu, TileConfig()).decode_tasks
    assert len(t54) == 216 and len(t55) == 220
    assert len(t55) - 2 * gpu.num_sms == 4
    assert all(t.op == 1 and not t.is_virtual and t.kv_split == (0, 16384) for t in t54)


def test_virtual_decode_subdivides():  # :62-84
    cfg = TileConfig(virtual_decode=True)
    wd = decompose_hybrid(decode_batch(1, 1000), GpuSpec.reference_default(), cfg)
    assert len(wd.decode_tasks) == 16
    assert all(t.is_virtual and t.slot_quanta == 1 for t in wd.decode_tasks)
    parents = decompose_hybrid(decode_batch(1, 1000), GpuSpec.reference_default(), TileConfig()).decode_tasks
    assert math.isclose(sum(t.compute_work for t in wd.decode_tasks), sum(t.compute_work for t in parents))
    assert math.isclose(sum(t.memory_work for t in wd.decode_tasks), sum(t.memory_work for t in parents))
    assert sum(t.kv_split[1] - t.kv_split[0] for t in wd.decode_tasks) == 4 * 1000


def test_limit_prefill_splits():  # :86-102
    gpu, cfg = GpuSpec.reference_default(), TileConfig()
    assert limit_prefill_splits(16, gpu, cfg) == 13
    assert limit_prefill_splits(216, gpu, cfg) == 1
    assert limit_prefill_splits(500, gpu, cfg) == 1
    assert limit_prefill_splits(1, gpu, cfg) == 216
    for par in (1, 2, 3, 5, 16, 31, 100, 215, 216, 217, 1000):
        best = max(s for s in range(1, 2 * gpu.num_sms + 1) if par * s <= 2 * gpu.num_sms or s == 1)
        assert limit_prefill_splits(par, gpu, cfg) == best
    with pytest.raises(InvalidArgument):
        limit_prefill_splits(0, gpu, cfg)


def test_prefill_decomposition_counts():  # :104-132
    gpu = GpuSpec.reference_default()
    b = HybridBatchSpec(prefill=PrefillSpec(512, 512, 0), shape=YI)
    assert len(decompose_hybrid(b, gpu, TileConfig(prefill_tile_q=128, split_wave_cap=0)).prefill_tasks) == 16
    b = HybridBatchSpec(prefill=PrefillSpec(16384, 16384, 0), shape=YI)
    assert len(decompose_hybrid(b, gpu, TileConfig()).prefill_tasks) == 512
    b = HybridBatchSpec(prefill=PrefillSpec(512, 16384, 15872), shape=YI)
    assert len(decompose_hybrid(b, gpu, TileConfig()).prefill_tasks) == 4 * 4 * 13


def test_prefill_kv_bytes_constant_across_split_caps():  # :134-176
    gpu = GpuSpec.reference_default()
    b = HybridBatchSpec(prefill=PrefillSpec(1024, 16384, 15360), shape=YI)
    prev = -1.0
    for cap in range(1, 5):
        cfg = TileConfig(split_wave_cap=cap)
        q_tiles = math.ceil(1024 / cfg.prefill_tile_q)
        splits = limit_prefill_splits(q_tiles * YI.num_kv_heads, gpu, cfg)
        tasks = decompose_hybrid(b, gpu, cfg).prefill_tasks
        kv = sum(2.0 * (t.kv_split[1] - t.kv_split[0]) * 128 for t in tasks)
        qb = sum(t.memory_work - 2.0 * (t.kv_split[1] - t.kv_split[0]) * 128 for t in tasks)
        exp_kv = sum(2.0 * (15360 + tile * 128 + 128) * 128 * 4 for tile in range(q_tiles))
        exp_q = sum(128.0 * 8 * 128 * 4 * splits for _ in range(q_tiles))
        assert math.isclose(kv, exp_kv, rel_tol=1e-12) and math.isclose(qb, exp_q, rel_tol=1e-12)
        assert kv + qb > prev
        prev = kv + qb


def test_select_tile_config():  # :178-209
    gpu = GpuSpec.reference_default()
    b = HybridBatchSpec(prefill=PrefillSpec(16384, 16384, 0), decodes=[DecodeSpec(12288)] * 64, shape=LLAMA_TP2)
    c = select_tile_config(b, gpu)
    assert (c.ctas_per_sm, c.prefill_tile_q, c.decode_tile_q) == (2, 128, 16)
    b = HybridBatchSpec(prefill=PrefillSpec(1024, 12288, 11264), decodes=[DecodeSpec(12288)] * 80, shape=LLAMA_TP2)
    c = select_tile_config(b, gpu)
    assert (c.ctas_per_sm, c.prefill_tile_q, c.decode_tile_q) == (4, 64, 16)
    c = select_tile_config(decode_batch(32, 8192, LLAMA_TP2), gpu)
    assert c.ctas_per_sm == 4
    assert decompose_hybrid(decode_batch(32, 8192, LLAMA_TP2), gpu).prefill_tasks == []


def test_make_tile_config():  # work_decomp.hpp:119-136
    c2, c4 = make_tile_config(2), make_tile_config(4)
    assert (c2.prefill_tile_q, c2.tile_kv, c2.shared_mem_per_cta) == (128, 64, 65536.0)
    assert (c4.prefill_tile_q, c4.tile_kv, c4.shared_mem_per_cta) == (64, 32, 32768.0)
    with pytest.raises(InvalidArgument):
        make_tile_config(3)


def test_hybrid_is_sum_of_parts():  # :211-244
    gpu = GpuSpec.reference_default()
    b = HybridBatchSpec(prefill=PrefillSpec(1536, 12288, 6144), decodes=[DecodeSpec(12288)] * 27, shape=YI)
    cfg = select_tile_config(b, gpu)
    wd = decompose_hybrid(b, gpu, cfg)
    only_p = HybridBatchSpec(prefill=b.prefill, shape=YI)
    only_d = HybridBatchSpec(decodes=b.decodes, shape=YI)
    assert wd.total_tasks() == len(decompose_hybrid(only_p, gpu, cfg).prefill_tasks) + \
        len(decompose_hybrid(only_d, gpu, cfg).decode_tasks)
    q_tiles = math.ceil(1536 / cfg.prefill_tile_q)
    splits = limit_prefill_splits(q_tiles * 4, gpu, cfg)
    assert len(wd.prefill_tasks) == q_tiles * 4 * splits
    assert len(wd.decode_tasks) == 27 * 4


def test_decode_count_invariant_random():  # :266-278
    rng = random.Random(17)
    for _ in range(50):
        kv = rng.randint(1, 8)
        shape = ModelShape(kv * rng.randint(1, 4), kv, 64, 8.0)
        n = rng.randint(1, 100)
        b = HybridBatchSpec(decodes=[DecodeSpec(rng.randint(1, 10000)) for _ in range(n)], shape=shape)
        assert len(decompose_hybrid(b, GpuSpec.reference_default(), TileConfig()).decode_tasks) == n * kv


def test_batch_validation():  # :293-302, work_decomp.hpp:33-47
    with pytest.raises(InvalidArgument):
        HybridBatchSpec(shape=YI).validate()
    with pytest.raises(InvalidArgument):
        HybridBatchSpec(prefill=PrefillSpec(1024, 512, 0), shape=YI).validate()
    with pytest.raises(InvalidArgument):
        HybridBatchSpec(decodes=[DecodeSpec(0)], shape=YI).validate()
    with pytest.raises(InvalidArgument):
        HybridBatchSpec(decodes=[DecodeSpec(8)], shape=ModelShape(6, 4, 128, 1.0)).validate()
    with pytest.raises(InvalidArgument):
        HybridBatchSpec(decodes=[DecodeSpec(8)], shape=ModelShape(8, 4, 128, 0.0)).validate()


# ------------------------------------ field-by-field vs compiled reference ---
def _random_batch(rng):
    kv = rng.choice([1, 2, 4, 8])
    shape = ModelShape(kv * rng.choice([1, 2, 4, 8]), kv, 128, rng.choice([11.3137, 8.0]))
    pf = None
    if rng.random() < 0.8:
        chunk = rng.randint(1, 4096)
        off = rng.randint(0, 20000)
        pf = PrefillSpec(chunk, off + chunk + rng.randint(0, 100), off)
    n = rng.randint(0 if pf else 1, 80)
    return HybridBatchSpec(prefill=pf, decodes=[DecodeSpec(rng.randint(1, 40000)) for _ in range(n)], shape=shape)


def _cmp(ours, theirs):
    assert len(ours) == len(theirs)
    for a, b in zip(ours, theirs):
        assert (a.op, a.request_id, a.kv_head, a.q_tile, a.kv_split, int(a.is_virtual), a.slot_quanta,
                a.barrier_segments) == (b.op, b.request_id, b.kv_head, b.q_tile, (b.kv_begin, b.kv_end),
                                        b.is_virtual, b.slot_quanta, b.barrier_segments)
        assert a.compute_work == b.compute_work and a.memory_work == b.memory_work  # bitwise doubles


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("gpu_name", ["reference", "b200"])
def test_task_table_matches_reference(gpu_name):
    gpu = GpuSpec.reference_default() if gpu_name == "reference" else GpuSpec.b200()
    rng = random.Random(2024 if gpu_name == "reference" else 7)
    for it in range(60):
        b = _random_batch(rng)
        shape = (b.shape.num_q_heads, b.shape.num_kv_heads, b.shape.head_dim, b.shape.scale)
        pf = (b.prefill.chunk_size, b.prefill.context_len, b.prefill.position_offset) if b.prefill else None
        ctx = [d.context_len for d in b.decodes]
        # (1) select_tile_config path
        st, rcfg, rp, rd = O.ref_decompose_hybrid(shape, pf, ctx, ref_gpu(gpu))
        assert st == 0
        wd = decompose_hybrid(b, gpu)
        assert (wd.config.ctas_per_sm, wd.config.prefill_tile_q, wd.config.tile_kv) == \
            (rcfg.ctas_per_sm, rcfg.prefill_tile_q, rcfg.tile_kv)
        _cmp(wd.prefill_tasks, rp)
        _cmp(wd.decode_tasks, rd)
        # (2) explicit config, virtual decode on/off, random split cap
        cfg = TileConfig(prefill_tile_q=rng.choice([16, 32, 64, 128]), tile_kv=rng.choice([16, 32, 64]),
                         virtual_decode=rng.random() < 0.5, split_wave_cap=rng.randint(0, 4))
        st, _, rp, rd = O.ref_decompose_hybrid(shape, pf, ctx, ref_gpu(gpu), ref_cfg(cfg))
        assert st == 0
        wd = decompose_hybrid(b, gpu, cfg)
        _cmp(wd.prefill_tasks, rp)
        _cmp(wd.decode_tasks, rd)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_limit_prefill_splits_matches_reference():
    for sms in (108, 148, 132):
        gpu = GpuSpec(num_sms=sms)
        for cap in (0, 1, 2, 3):
            cfg = TileConfig(split_wave_cap=cap)
            for nat in (1, 2, 7, 64, 128, 148, 296, 1000):
                st, ref = O.ref_limit_prefill_splits(nat, ref_gpu(gpu), ref_cfg(cfg))
                assert st == 0 and limit_prefill_splits(nat, gpu, cfg) == ref


# --------------------------------------------------- scheduler semantics ---
def test_sm_aware_ticket_patterns():  # test_gpu_sim.cpp:80-114
    (pr, dr), ops, _ = O.sched_replay(0, 10, 10, 1, [0] * 4)
    assert list(ops) == [0, 1, 0, 1]
    (pr, dr), ops, _ = O.sched_replay(1, 50, 100, 1, [0] * 6)
    assert (pr, dr) == (1, 2) and list(ops) == [0, 1, 1, 0, 1, 1]
    _, ops, _ = O.sched_replay(0, 2, 6, 1, [0] * 9)
    assert list(ops[:8]).count(0) == 2 and all(o == 1 for o in ops[4:8]) and ops[8] == -1
    _, ops, ids = O.sched_replay(0, 3, 3, 2, [i % 2 for i in range(6)])
    assert [i for o, i in zip(ops, ids) if o == 0] == [0, 1, 2]
    assert [i for o, i in zip(ops, ids) if o == 1] == [0, 1, 2]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_scheduler_port_matches_reference_and_claims_once():
    rng = random.Random(5)
    for it in range(200):
        P, D = rng.randint(0, 40), rng.randint(0, 40)
        if P + D == 0:
            continue
        sms = rng.choice([1, 3, 7, 148])
        seq = [rng.randrange(sms) for _ in range(P + D)]
        for prop in (0, 1):
            a = O.sched_replay(prop, P, D, sms, seq, which="port")
            b = O.sched_replay(prop, P, D, sms, seq, which="ref")
            assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
            ops, ids = a[1], a[2]
            assert sorted(ids[ops == 0].tolist()) == list(range(P))
            assert sorted(ids[ops == 1].tolist()) == list(range(D))


def test_plan_ratio_policies():
    b = HybridBatchSpec(prefill=PrefillSpec(1024, 16384, 15360), decodes=[DecodeSpec(16384)] * 64,
                        shape=ModelShape(32, 8, 128, math.sqrt(128)))
    gpu = GpuSpec.b200()
    i = Plan(b, gpu, PlanOptions(policy=0)).info()
    assert (i.prefill_ratio, i.decode_ratio) == (1, 1)
    i = Plan(b, gpu, PlanOptions(policy=1)).info()
    g = math.gcd(i.num_prefill_ctas, i.num_decode_ctas)
    assert (i.prefill_ratio, i.decode_ratio) == (i.num_prefill_ctas // g, i.num_decode_ctas // g)
    i = Plan(b, gpu, PlanOptions(policy=2)).info()
    assert i.prefill_ratio + i.decode_ratio == max(2, i.config.ctas_per_sm) and i.prefill_ratio >= 1


def test_b200_plan_lowering():
    """B200 tile mode: one 128-row M-block per prefill item (two for the warp-
    specialised pair engine); decode items cover each (request, kv head) with
    4 virtual warps whose ranges are the reference's virtual tasks when
    decode_splits = 1."""
    from paper_2410_18038_b200._abi import POD_POLICY_FIFTY_FIFTY, POD_POLICY_WARPSPEC
    shape = ModelShape(32, 8, 128, math.sqrt(128))
    b = HybridBatchSpec(prefill=PrefillSpec(1024, 16384, 15360), decodes=[DecodeSpec(16384)] * 64, shape=shape)
    i = Plan(b, GpuSpec.b200(), PlanOptions(tile_mode=POD_TILE_B200, policy=POD_POLICY_FIFTY_FIFTY)).info()
    assert i.config.prefill_tile_q * shape.group_size() == 128
    assert i.num_prefill_ctas == i.num_prefill_tasks == 32 * 8 * i.prefill_splits
    p = Plan(b, GpuSpec.b200(), PlanOptions(tile_mode=POD_TILE_B200, decode_splits=1, policy=POD_POLICY_WARPSPEC))
    i = p.info()
    assert i.config.prefill_tile_q * shape.group_size() == 256
    assert i.num_prefill_ctas == i.num_prefill_tasks == 16 * 8 * i.prefill_splits
    assert i.num_decode_tasks == 64 * 8 * 4 and i.num_decode_ctas == 64 * 8
    wd = p.tasks()
    for t in wd.decode_tasks[:16]:
        assert t.is_virtual
    # the virtual ranges of parent (0, 0) are split_ranges(16384, 4)
    assert [t.kv_split for t in wd.decode_tasks[:4]] == pkg.split_ranges(16384, 4)


@pytest.mark.parametrize("policy", [4, 5, 6, 9, -1])
def test_retired_and_unknown_policies_are_rejected(policy):
    shape = ModelShape(32, 8, 128, math.sqrt(128))
    b = HybridBatchSpec(prefill=PrefillSpec(64, 128, 64), decodes=[DecodeSpec(100)], shape=shape)
    with pytest.raises(InvalidArgument, match="policy"):
        Plan(b, GpuSpec.b200(), PlanOptions(policy=policy))


def test_decode_split_count_per_request_is_clamped_to_context():
    """an explicit decode_splits larger than a request's context
    gives that request min(splits, ctx) CTAs; the plan's per-request counts (read by
    the merge) match the CTA table."""
    shape = ModelShape(32, 8, 128, math.sqrt(128))
    b = HybridBatchSpec(decodes=[DecodeSpec(1), DecodeSpec(3), DecodeSpec(2000)], shape=shape)
    for policy in (3, 7):
        p = Plan(b, GpuSpec.b200(), PlanOptions(policy=policy, decode_splits=4))
        i = p.info()
        assert i.num_decode_ctas == 8 * (1 + 3 + 4)
        assert i.num_merge_rows_decode == 2 * 32  # requests 1 and 2 merge, request 0 writes directly


def test_auto_engine_choice_and_v_shadow_workspace():
    """AUTO's measured engine rules at the BASELINE shapes (pod_plan.cpp):
    the 64-key pair engine below a decode share of 0.57, with two S buffers below 0.30, the
    32-key engine above; the fp16 V shadow (prefill V converted once per launch) for F16PV
    bf16 plans on the two-CTA kernel and the 64-key engine, sized [pages][Hkv][16][d] fp16."""
    from paper_2410_18038_b200._abi import POD_PRECISION_SPLIT, POD_POLICY_COMPLEMENT
    shape = ModelShape(32, 8, 128, math.sqrt(128))

    def c2(nb):
        return HybridBatchSpec(prefill=PrefillSpec(1024, 16384, 15360), decodes=[DecodeSpec(16384)] * nb,
                               shape=shape)

    want = {8: (64, 2), 16: (64, 2), 32: (64, 1), 64: (32, 2)}  # decode share 0.17 / 0.29 / 0.45 / 0.62
    for nb, (keys, sb) in want.items():
        i = Plan(c2(nb), GpuSpec.b200()).info()
        assert (i.prefill_tile_keys, i.prefill_s_buffers) == (keys, sb), nb
    c1 = HybridBatchSpec(prefill=PrefillSpec(512, 2048, 1536), decodes=[DecodeSpec(2048)] * 8, shape=shape)
    assert (Plan(c1, GpuSpec.b200()).info().prefill_tile_keys, Plan(c1, GpuSpec.b200()).info().prefill_s_buffers) == (64, 1)
    # the shadow: 16384 keys = 1024 logical pages x 8 KV heads x 16 x 128 x 2 B = 32 MiB of workspace
    shadow = 1024 * 8 * 16 * 128 * 2
    ws = {}
    for name, opts in (("complement", PlanOptions(policy=POD_POLICY_COMPLEMENT)),
                       ("complement_split", PlanOptions(policy=POD_POLICY_COMPLEMENT, precision=POD_PRECISION_SPLIT)),
                       ("ws32", PlanOptions(prefill_tile_keys=32)), ("ws64", PlanOptions(prefill_tile_keys=64))):
        ws[name] = Plan(c2(64), GpuSpec.b200(), opts).workspace_bytes()
    assert ws["complement"] - ws["complement_split"] >= shadow  # F16PV adds the shadow, SPLIT does not
    assert ws["ws64"] - ws["ws32"] >= shadow - (1 << 20)        # 64-key plans carry it, 32-key ones do not


def test_tuned_options_signature_buckets():
    """tune.TunedOptions memoises per bucketed batch signature: decode contexts and the
    prefill offset round up to the bucket, so nearby serving-loop shapes share one search."""
    from paper_2410_18038_b200.tune import TunedOptions, default_candidates
    shape = ModelShape(32, 8, 128, math.sqrt(128))
    t = TunedOptions(bucket=256)
    a = HybridBatchSpec(prefill=PrefillSpec(256, 2048, 1792), decodes=[DecodeSpec(2048)] * 4, shape=shape)
    b = HybridBatchSpec(prefill=PrefillSpec(256, 1956, 1700), decodes=[DecodeSpec(2000)] * 4, shape=shape)
    c = HybridBatchSpec(prefill=PrefillSpec(256, 2300, 2044), decodes=[DecodeSpec(2300)] * 4, shape=shape)
    assert t.signature(a) == t.signature(b) != t.signature(c)
    names = [n for n, _ in default_candidates(a)]
    assert names[0] == "auto" and "warpspec/64-key/double-S" in names and len(names) == len(set(names))
    assert [n for n, _ in default_candidates(HybridBatchSpec(decodes=[DecodeSpec(100)], shape=shape))][0] == "auto"
