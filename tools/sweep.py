#!/usr/bin/env python3
"""C5 sweep (BASELINE.json configs[4]): prefill chunk x context x decode batch,
fused vs serial vs the combined roofline, on one B200 (Llama-3-8B shape, AUTO policy).
Each point: synthetic bf16 inputs resident in HBM, L2 flushed before every timed
run, median of `--reps` CUDA-event timings.  Prints one JSON line per point.

  python tools/sweep.py [--chunks 512,1024,2048,4096] [--ctx 4096,16384,65536] [--batches 8,64,256]
"""
import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2410_18038_b200 as pkg  # noqa: E402
from bench import peaks, work  # noqa: E402
from paper_2410_18038_b200.hybrid import PodAttention  # noqa: E402
from paper_2410_18038_b200.workload import build_workload, make_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", default="512,1024,2048,4096")
    ap.add_argument("--ctx", default="4096,16384,65536")
    ap.add_argument("--batches", default="8,64,256")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--max-kv-gb", type=float, default=80.0)
    ap.add_argument("--policy", type=int, default=8, help="POD_POLICY_* (8 = AUTO)")
    ap.add_argument("--heads", default="32,8", help="q heads, kv heads")
    a = ap.parse_args()
    pk = peaks()
    hq, hkv = map(int, a.heads.split(","))
    shape = pkg.ModelShape(hq, hkv, 128, math.sqrt(128))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for ctx in map(int, a.ctx.split(",")):
        for b in map(int, a.batches.split(",")):
            kv_gb = b * ctx * hkv * 128 * 4 / 1e9
            if kv_gb > a.max_kv_gb:
                print(json.dumps({"ctx": ctx, "batch": b, "skipped": f"{kv_gb:.0f} GB of KV"}))
                continue
            for chunk in map(int, a.chunks.split(",")):
                off = ctx - chunk
                batch = make_batch(shape, chunk=chunk, offset=off, decode_ctx=[ctx] * b)
                wl = build_workload(batch, device="cuda")
                op = PodAttention(batch, options=pkg.PlanOptions(policy=a.policy))
                out = op.alloc_outputs()
                res = {}
                for mode in ("fused", "serial", "prefill", "decode"):
                    for _ in range(2):
                        op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices,
                               out=out, mode=mode)
                    ts = []
                    for _ in range(a.reps):
                        flush.zero_()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices,
                               out=out, mode=mode)
                        e1.record()
                        ts.append((e0, e1))
                    torch.cuda.synchronize()
                    v = sorted(x.elapsed_time(y) * 1000 for x, y in ts)
                    res[mode] = v[len(v) // 2]
                flops, dbytes = work(32, 8, chunk, off, b, ctx)
                roof = max(flops / (pk["bf16_tflops"] * 1e12), dbytes / (pk["hbm_gbs"] * 1e9)) * 1e6
                print(json.dumps({"chunk": chunk, "ctx": ctx, "batch": b, "policy": {3: "complement", 7: "warpspec"}.get(
                    op.info.policy, op.info.policy), "fused_us": round(res["fused"], 1), "serial_us": round(res["serial"], 1),
                    "prefill_us": round(res["prefill"], 1), "decode_us": round(res["decode"], 1),
                    "speedup": round(res["serial"] / res["fused"], 3),
                    "fused_vs_max_alone": round(res["fused"] / max(res["prefill"], res["decode"]), 3),
                    "roofline_us": round(roof, 1), "roofline_frac": round(roof / res["fused"], 3)}), flush=True)
                op.plan.close()
                del wl, op, out
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
