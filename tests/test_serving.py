"""Serving-loop caller: the Python restatement of the reference's
request-level simulator (serving.hpp) is pinned against the reference compiled in
place (oracle/_ref): identical traces, identical iteration records and metrics under
the linear cost the reference's own serving tests use (test_serving.cpp)."""
import math

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2410_18038_b200.pod import DecodeSpec, HybridBatchSpec, ModelShape, PrefillSpec
from paper_2410_18038_b200.serving import (Request, SchedulerPolicy, TokenDist, generate_trace, percentile,
                                           run_serving)
from paper_2410_18038_b200.workload import Rng

SHAPE = ModelShape(16, 4, 128, 11.3137)
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def linear(c0, c1):
    def cost(batch, fused):
        tokens = batch.prefill.chunk_size if batch.prefill is not None else 0
        return c0 + c1 * (tokens + len(batch.decodes))
    return cost


def test_percentile_nearest_rank():  # test_serving.cpp:27-48
    v = list(range(1, 101))
    assert percentile(v, 50) == 50 and percentile(v, 99) == 99 and percentile(v, 100) == 100
    assert percentile(v, 0) == 1
    with pytest.raises(ValueError):
        percentile([], 50)
    rng = Rng(5)
    for _ in range(50):
        n = rng.next_long(1, 40)
        s = [float(rng.next_long(0, 10)) for _ in range(n)]
        p = float(rng.next_long(0, 100))
        rank = max(1, math.ceil(p / 100.0 * n))
        assert percentile(s, p) == sorted(s)[rank - 1]


@needs_ref
@pytest.mark.parametrize("dists", [(TokenDist("uniform", 512, 2048), TokenDist("uniform", 16, 128)),
                                   (TokenDist("lognormal", 7.0, 0.5), TokenDist("fixed", 64, 0)),
                                   (TokenDist("fixed", 1024, 0), TokenDist("lognormal", 4.0, 1.0))])
def test_trace_generation_equals_reference(dists):
    pd, dd = dists
    ours = generate_trace(1.5, 200, pd, dd, 99)
    arr, pt, dt = O.ref_generate_trace(1.5, 200, pd, dd, 99)
    assert [r.arrival_time for r in ours] == arr.tolist()
    assert [r.prefill_tokens for r in ours] == pt.tolist()
    assert [r.decode_tokens for r in ours] == dt.tolist()


def _offline(n, prefill, decode):
    return [Request(0.0, prefill, decode) for _ in range(n)]


@needs_ref
@pytest.mark.parametrize("policy", [SchedulerPolicy.prefill_prioritized(), SchedulerPolicy.chunked_hybrid(512),
                                    SchedulerPolicy.chunked_hybrid(1024, max_batch=16, token_budget=1100),
                                    SchedulerPolicy.chunked_hybrid(2048)])
def test_run_serving_equals_reference(policy):
    traces = [generate_trace(0.02, 60, TokenDist("uniform", 300, 3000), TokenDist("uniform", 5, 80), 7),
              _offline(24, 1500, 37)]
    traces[1][3].prefill_tokens = 700
    traces[1][9].prefill_tokens = 2049
    for trace in traces:
        res = run_serving(trace, policy, linear(1.0, 0.001), False, SHAPE)
        its, ttft, lat, met = O.ref_run_serving_linear(trace, policy, 1.0, 0.001)
        got = [(r.t_start, r.t_end, r.prefill_request, r.prefill_tokens, r.decode_requests) for r in res.iterations]
        assert got == [(a, b, int(c), int(d), int(e)) for a, b, c, d, e in its]
        assert res.ttft == ttft.tolist() and res.latency == lat.tolist()
        m = res.metrics
        assert [m.ttft_p50, m.ttft_p99, m.tbt_p50, m.tbt_p99, m.latency_p50, m.latency_p99, m.throughput,
                m.stall_pct_at[0][1], m.stall_pct_at[1][1]] == met.tolist()


def test_token_conservation_and_no_decode_pause():  # test_serving.cpp:113-133
    trace = _offline(24, 1500, 37)
    trace[3].prefill_tokens = 700
    trace[9].prefill_tokens = 2049
    res = run_serving(trace, SchedulerPolicy.chunked_hybrid(512), linear(1.0, 0.001), False, SHAPE)
    sums = [0] * len(trace)
    for it in res.iterations:
        if it.prefill_request >= 0:
            sums[it.prefill_request] += it.prefill_tokens
    assert sums == [r.prefill_tokens for r in trace]
    assert [len(v) for v in res.tbt] == [r.decode_tokens for r in trace]


def test_steady_state_hybrid_batch():  # test_serving.cpp:92-111
    res = run_serving(_offline(200, 2048, 200), SchedulerPolicy.chunked_hybrid(1024), linear(1.0, 0.001), False,
                      SHAPE)
    best = streak = 0
    for it in res.iterations:
        streak = streak + 1 if (it.prefill_request >= 0 and it.decode_requests == 100) else 0
        best = max(best, streak)
    assert best >= 100


def test_single_request_policies_coincide():  # test_serving.cpp:81-90
    trace = _offline(1, 2048, 20)
    pp = run_serving(trace, SchedulerPolicy.prefill_prioritized(), linear(5.0, 0.01), False, SHAPE)
    ch = run_serving(trace, SchedulerPolicy.chunked_hybrid(2048), linear(5.0, 0.01), False, SHAPE)
    assert pp.metrics.ttft_p50 == ch.metrics.ttft_p50 and pp.metrics.tbt_p99 == ch.metrics.tbt_p99
    assert len(pp.iterations) == len(ch.iterations)


def test_invalid_inputs():
    with pytest.raises(ValueError):
        run_serving([], SchedulerPolicy.chunked_hybrid(512), linear(1, 0), False, SHAPE)
    with pytest.raises(ValueError):
        run_serving([Request(1.0), Request(0.5)], SchedulerPolicy.chunked_hybrid(512), linear(1, 0), False, SHAPE)
    with pytest.raises(ValueError):
        generate_trace(0.0, 3, TokenDist(), TokenDist(), 1)


@pytest.mark.gpu
def test_measured_cost_serving_fused_vs_serial():
    """The attention term measured on the B200 (pod_attn_run vs pod_attn_run_serial):
    hybrid iterations are cheaper fused, decode-only ones are not slower, and the
    fused serving run's TBT p50 is no worse than the serial one's."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs cuda:0")
    from paper_2410_18038_b200.serving import MeasuredIterationCost

    shape = ModelShape(32, 8, 128, math.sqrt(128))
    cost = MeasuredIterationCost(shape, bucket=1024, repeats=3)
    hyb = HybridBatchSpec(prefill=PrefillSpec(512, 8192, 4096), decodes=[DecodeSpec(8192)] * 16, shape=shape)
    assert cost(hyb, True) < cost(hyb, False)
    trace = generate_trace(0.02, 12, TokenDist("uniform", 1024, 4096), TokenDist("uniform", 8, 24), 3)
    f = run_serving(trace, SchedulerPolicy.chunked_hybrid(512), cost, True, shape)
    s = run_serving(trace, SchedulerPolicy.chunked_hybrid(512), cost, False, shape)
    assert f.metrics.tbt_p50 <= s.metrics.tbt_p50 * 1.05
    assert all(np.isfinite(f.ttft)) and f.metrics.ttft_p99 > 0
