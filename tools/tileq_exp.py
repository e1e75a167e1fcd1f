"""C1 / TP-rank shapes: the warp-specialised kernel with single-block prefill items
(prefill_tile_q = 128 / G: no KV split needed for C1) vs the default pair items.

  python tools/tileq_exp.py
"""
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


def timeit(op, wl, mode, flush, n=20):
    out = op.alloc_outputs()

    def step():
        op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, out=out, mode=mode)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        flush.zero_()
        a.record()
        step()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) * 1000 for a, b in ev)
    return ms[n // 2]


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for cfg in ("c1", "c3_tp8_rank", "c3_tp4_rank", "c2_b8"):
        hq, hkv, chunk, off, b, ctx = CONFIGS[cfg]
        G = hq // hkv
        batch = make_batch(pkg.ModelShape(hq, hkv, 128, math.sqrt(128)), chunk=chunk, offset=off, decode_ctx=[ctx] * b)
        wl = build_workload(batch, device="cuda")
        for name, opts in (("auto", pkg.PlanOptions()),
                           ("single-block", pkg.PlanOptions(policy=7, tile_override=pkg.TileConfig(
                               prefill_tile_q=128 // G, tile_kv=64, split_wave_cap=1, virtual_decode=True))),
                           ("single-block cap2", pkg.PlanOptions(policy=7, tile_override=pkg.TileConfig(
                               prefill_tile_q=128 // G, tile_kv=64, split_wave_cap=2, virtual_decode=True)))):
            try:
                op = PodAttention(batch, options=opts)
            except Exception as e:  # noqa: BLE001
                print(cfg, name, "plan failed", e)
                continue
            i = op.info
            r = {m: timeit(op, wl, m, flush) for m in ("fused", "prefill")}
            print(f"{cfg:12s} {name:18s} fused {r['fused']:7.1f} prefill {r['prefill']:7.1f} us | items {i.num_prefill_ctas}"
                  f"/{i.num_decode_ctas} splits {i.prefill_splits} merges {i.num_merge_rows_prefill}/{i.num_merge_rows_decode}"
                  f" keys {i.prefill_tile_keys}")


if __name__ == "__main__":
    main()
