"""Extended GPU fuzz: cases 48..N of tests/test_gpu_fuzz.py's generator (every kernel in turn,
head dims 32/64/128, peaky queries), each against the dense float64 layer.

    python tools/fuzz_more.py [N]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2410_18038_b200 as pkg  # noqa: E402
from paper_2410_18038_b200.hybrid import PodAttention  # noqa: E402
from paper_2410_18038_b200.tp import layer_error  # noqa: E402
from paper_2410_18038_b200.workload import build_workload, make_batch  # noqa: E402
from tests.common import LSE_TOL, O_TOL, dense_layer  # noqa: E402
from tests.test_gpu_fuzz import _case  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    bad = 0
    worst = 0.0
    for i in range(48, n):
        shape, chunk, offset, ctx, q_scale, name, opts = _case(i)
        batch = make_batch(shape, chunk=chunk, offset=offset, decode_ctx=ctx)
        wl = build_workload(batch, device="cuda", q_scale=q_scale, seed_q=42 + i, seed_kv=43 + i)
        try:
            op = PodAttention(batch, options=pkg.PlanOptions(**opts))
        except pkg.Unsupported:
            continue
        out = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)
        torch.cuda.synchronize()
        o = torch.cat([t for t in (out.o_prefill, out.o_decode) if t is not None])
        lse = torch.cat([t for t in (out.lse_prefill, out.lse_decode) if t is not None])
        o_ref, lse_ref = dense_layer(wl)
        eo, el = layer_error(o, lse, o_ref, lse_ref, shape.group_size())
        worst = max(worst, eo)
        if not (torch.isfinite(o).all() and eo <= O_TOL and el <= LSE_TOL):
            bad += 1
            print("FAIL", i, name, shape, chunk, offset, ctx[:4], q_scale, eo, el, flush=True)
    print(f"fuzz {48}..{n}: {bad} failures, worst O error {worst:.2e}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
