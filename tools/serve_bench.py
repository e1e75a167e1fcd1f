#!/usr/bin/env python3
"""Serving-loop benchmark: the reference's request-level loop
(paper_2410_18038_b200/serving.py, pinned to serving.hpp) with the attention term
of every iteration measured on the B200 (fused pod_attn_run vs serial), for a
Llama-3-8B-shaped model (32 attention layers).  Prints one JSON line.

  python tools/serve_bench.py [--qps 0.5] [--requests 48] [--chunk 1024]
"""
import argparse
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2410_18038_b200.pod import ModelShape  # noqa: E402
from paper_2410_18038_b200.serving import (MeasuredIterationCost, SchedulerPolicy, TokenDist,  # noqa: E402
                                           generate_trace, run_serving)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qps", type=float, default=2.0, help="arrivals per second")
    ap.add_argument("--requests", type=int, default=48)
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--w-fixed", type=float, default=0.0, help="us per iteration outside attention")
    ap.add_argument("--w-tok", type=float, default=0.0, help="us per token outside attention")
    a = ap.parse_args()
    shape = ModelShape(32, 8, 128, math.sqrt(128))
    trace = generate_trace(a.qps / 1e6, a.requests, TokenDist("uniform", 4096, 16384), TokenDist("uniform", 64, 512), 11)
    cost = MeasuredIterationCost(shape, w_fixed=a.w_fixed, w_tok=a.w_tok, bucket=512, repeats=3, layers=a.layers)
    out = {"metric": "serving TTFT / TBT with measured B200 attention", "unit": "us", "layers": a.layers,
           "trace": {"requests": a.requests, "qps": a.qps, "prefill": "uniform 4096-16384",
                     "decode": "uniform 64-512", "chunk": a.chunk}}
    t0 = time.time()
    for fused in (True, False):
        r = run_serving(trace, SchedulerPolicy.chunked_hybrid(a.chunk), cost, fused, shape)
        m = r.metrics
        out["fused" if fused else "serial"] = {
            "ttft_p50": round(m.ttft_p50, 1), "ttft_p99": round(m.ttft_p99, 1), "tbt_p50": round(m.tbt_p50, 1),
            "tbt_p99": round(m.tbt_p99, 1), "latency_p99": round(m.latency_p99, 1),
            "throughput_rps": round(m.throughput * 1e6, 3), "iterations": len(r.iterations)}
    out["measured_shapes"] = cost.measurements
    out["wall_s"] = round(time.time() - t0, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
