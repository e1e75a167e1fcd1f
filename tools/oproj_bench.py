"""o_proj consumer timing: pod_oproj_run (tcgen05 GEMM, store or reduce-scatter epilogue)
vs torch.matmul (cuBLAS) on the Llama-3-8B layer shape (tokens = 1024 + 64, K = Hq/T x 128,
N = hidden 4096), L2 flushed between runs.

  python tools/oproj_bench.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2410_18038_b200.tp import oproj  # noqa: E402


def timeit(fn, flush, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) * 1000 for a, b in ev)
    return ms[n // 2]


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    tokens, n = 1088, 4096
    for t in (1, 2, 4, 8):
        k = 4096 // t
        o = (torch.rand(tokens, k, device="cuda") * 2 - 1).to(torch.bfloat16)
        w = ((torch.rand(k, n, device="cuda") * 2 - 1) / 64).to(torch.bfloat16)
        y = torch.empty(tokens, n, device="cuda")
        rows = (tokens + t - 1) // t
        ys = [torch.zeros(rows, n, device="cuda") for _ in range(t)]
        flops = 2.0 * tokens * k * n
        us_store = timeit(lambda: oproj(o, w, [y]), flush)
        us_red = timeit(lambda: oproj(o, w, ys, rows_per_rank=rows, accumulate=True), flush)
        us_torch = timeit(lambda: torch.matmul(o, w, out=None), flush)
        print(f"TP{t}: K={k}: pod_oproj store {us_store:.1f} us ({flops / us_store / 1e6:.0f} TF/s), "
              f"reduce-scatter epilogue {us_red:.1f} us, torch.matmul bf16->bf16 {us_torch:.1f} us "
              f"({flops / us_torch / 1e6:.0f} TF/s)")


if __name__ == "__main__":
    main()
