"""Max prefill / decode error vs the CPU oracle for each P precision mode
(test infrastructure: uses oracle/ as the checker)."""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2410_18038_b200 as pkg  # noqa: E402
from paper_2410_18038_b200.hybrid import PodAttention  # noqa: E402
from paper_2410_18038_b200.workload import build_workload, make_batch  # noqa: E402
from tests.common import compare_decode, compare_prefill  # noqa: E402

shape = pkg.ModelShape(32, 8, 128, math.sqrt(128))
cases = [("c2-like 16K", dict(chunk=128, offset=16256, decode_ctx=[16384] * 2), [(0, 8), (120, 128)]),
         ("2K", dict(chunk=512, offset=1536, decode_ctx=[2048] * 4), [(0, 512)]),
         ("short", dict(chunk=256, offset=0, decode_ctx=[100, 17]), [(0, 256)])]
for name, kw, rows in cases:
    batch = make_batch(shape, **kw)
    for q_scale in (1.0, 8.0):
        wl = build_workload(batch, device="cuda", q_scale=q_scale)
        for prec in (0, 1):
            op = PodAttention(batch, options=pkg.PlanOptions(precision=prec))
            out = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)
            torch.cuda.synchronize()
            o, l = out.o_prefill.cpu().numpy(), out.lse_prefill.cpu().numpy()
            eo = max(compare_prefill(wl, o, l, kv_heads=[0, 5], row_range=r)[0] for r in rows)
            do, _ = compare_decode(wl, out.o_decode.cpu().numpy(), out.lse_decode.cpu().numpy(), requests=[0])
            print(f"{name:12s} q*{q_scale:3.0f} precision {prec}: prefill O rel err {eo:.2e}   decode {do:.2e}")
