"""Eager (Python -> ctypes -> pod_attn_run per step) vs CUDA-graph replay of the same
fused layer, L2 flushed between steps: separates host launch overhead from device time.

  python tools/graph_vs_eager.py --config c1
"""
import argparse
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2410_18038_b200 as pkg  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2410_18038_b200.hybrid import PodAttention  # noqa: E402
from paper_2410_18038_b200.workload import build_workload, make_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--mode", default="fused")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    hq, hkv, chunk, off, b, ctx = CONFIGS[a.config]
    batch = make_batch(pkg.ModelShape(hq, hkv, 128, math.sqrt(128)), chunk=chunk, offset=off, decode_ctx=[ctx] * b)
    wl = build_workload(batch, device="cuda")
    op = PodAttention(batch)
    out = op.alloc_outputs()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def step():
        op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, out=out, mode=a.mode)

    from paper_2410_18038_b200.hybrid import l2_flush

    def timed(fn, flush_between=True, own_flush=False):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
        for e0, e1 in ev:
            if flush_between and own_flush:
                l2_flush(flush)
            elif flush_between:
                flush.zero_()
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        ms = sorted(x.elapsed_time(y) * 1000 for x, y in ev)
        return ms[len(ms) // 2], ms[0]

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    e_med, e_min = timed(step)
    g_med, g_min = timed(g.replay)
    e2_med, _ = timed(step, flush_between=False)
    e3_med, _ = timed(step, own_flush=True)
    print(f"{a.config} {a.mode}: eager median {e_med:.1f} (min {e_min:.1f}) us | graph median {g_med:.1f} "
          f"(min {g_min:.1f}) us | eager, no flush {e2_med:.1f} us | eager, pod_attn_l2_flush {e3_med:.1f} us | plan items {op.info.num_prefill_ctas}"
          f"/{op.info.num_decode_ctas} merges {op.info.num_merge_rows_prefill}/{op.info.num_merge_rows_decode}")


if __name__ == "__main__":
    main()
