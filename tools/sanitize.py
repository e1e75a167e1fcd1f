"""Small hybrid batches through every POD kernel path, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py

Covers the warp-specialised kernel (both pair-engine tile widths, also on a 3-CTA grid
where every CTA runs several prefill items back to back), the two-CTA
kernel, the decode split merge, the prefill split merge, serial mode, and the
KV append.  Outputs are checked loosely (finite) -- parity is the test suite's job;
this script only drives the kernels under the sanitizer.
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2410_18038_b200 as pkg  # noqa: E402
from paper_2410_18038_b200._abi import POD_POLICY_COMPLEMENT, POD_POLICY_WARPSPEC  # noqa: E402
from paper_2410_18038_b200.hybrid import PodAttention  # noqa: E402
from paper_2410_18038_b200.workload import build_workload, make_batch  # noqa: E402


def run(batch, opts, modes=("fused",), nsm=0):
    import dataclasses

    wl = build_workload(batch, device="cuda")
    gpu = pkg.GpuSpec.from_device(0)
    if nsm:  # a small grid: every CTA runs several items back to back (ring / epilogue-tile reuse)
        gpu = dataclasses.replace(gpu, num_sms=nsm)
    op = PodAttention(batch, gpu=gpu, options=opts)
    for mode in modes:
        out = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, mode=mode)
        torch.cuda.synchronize()
        for t in (out.o_prefill, out.o_decode):
            if t is not None:
                assert torch.isfinite(t.float()).all()
    info = op.info
    print(f"ok policy={info.policy} tile_keys={getattr(info, 'prefill_tile_keys', '?')} "
          f"pctas={info.num_prefill_ctas} dctas={info.num_decode_ctas} modes={modes}", flush=True)


def main():
    shape = pkg.ModelShape(32, 8, 128, 128 ** 0.5)
    small = make_batch(shape, chunk=128, offset=448, decode_ctx=[512, 300, 17, 1])
    cases = [
        (small, pkg.PlanOptions(policy=POD_POLICY_WARPSPEC), ("fused", "serial")),
        (small, pkg.PlanOptions(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=64), ("fused",)),
        (small, pkg.PlanOptions(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=64, prefill_s_buffers=2), ("fused", "serial")),
        (small, pkg.PlanOptions(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=32, decode_splits=3), ("fused",)),
        (small, pkg.PlanOptions(policy=POD_POLICY_COMPLEMENT, split_wave_cap=4, decode_splits=2), ("fused", "serial")),
    ]
    for batch, opts, modes in cases:
        run(batch, opts, modes)
    d64 = make_batch(pkg.ModelShape(16, 4, 64, 8.0), chunk=100, offset=300, decode_ctx=[500, 33, 1])
    run(d64, pkg.PlanOptions(policy=POD_POLICY_WARPSPEC), ("fused",))  # head dim 64, zero-padded
    run(d64, pkg.PlanOptions(policy=POD_POLICY_COMPLEMENT, decode_splits=2), ("fused",))
    many = make_batch(shape, chunk=256, offset=200, decode_ctx=[300, 64, 5])
    for keys, sb in ((32, 0), (64, 1), (64, 2)):
        run(many, pkg.PlanOptions(policy=POD_POLICY_WARPSPEC, prefill_tile_keys=keys, prefill_s_buffers=sb), ("fused",),
            nsm=3)
    # the o_proj consumer: store and reduce-scatter epilogues (virtual ranks)
    from paper_2410_18038_b200.tp import oproj
    o = (torch.rand(200, 512, device="cuda") - 0.5).to(torch.bfloat16)
    w = (torch.rand(512, 256, device="cuda") - 0.5).to(torch.bfloat16)
    oproj(o, w, [torch.empty(200, 256, device="cuda")])
    ys = [torch.zeros(100, 256, device="cuda") for _ in range(2)]
    for r in range(2):
        oproj(o[:, 256 * r:256 * (r + 1)].contiguous(), w[256 * r:256 * (r + 1)].contiguous(), ys, rows_per_rank=100,
              accumulate=True)
    torch.cuda.synchronize()
    print("ok o_proj")
    print("sanitize driver done")


if __name__ == "__main__":
    main()
