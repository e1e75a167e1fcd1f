"""Measured kernel selection (paper_2410_18038_b200/tune.py): the search the reference
runs on its simulator (best_fused_makespan, gpu_sim.hpp:802-816), on the hardware.
The tuned options must run the batch correctly (oracle parity) and be no slower than
the AUTO plan beyond timing noise; the memo must return the same choice per bucketed
signature."""
import math

import pytest
import torch

import paper_2410_18038_b200 as pkg
from paper_2410_18038_b200.tune import TunedOptions, tune_options
from paper_2410_18038_b200.workload import build_workload, make_batch
from tests.common import LSE_TOL, O_TOL, compare_decode, compare_prefill

pytestmark = pytest.mark.gpu


def test_tuned_options_are_fastest_and_correct():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2410_18038_b200.hybrid import PodAttention

    batch = make_batch(pkg.ModelShape(32, 8, 128, math.sqrt(128)), chunk=256, offset=1792, decode_ctx=[2048] * 16)
    wl = build_workload(batch, device="cuda")
    best, table = tune_options(batch, workload=wl, reps=5)
    names = [n for n, _ in table]
    assert "auto" in names and len(table) >= 4
    auto_us = dict(table)["auto"]
    assert table[0][1] <= auto_us  # the winner is at least as fast as AUTO
    out = PodAttention(batch, options=best).run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr,
                                                wl.page_indices)
    torch.cuda.synchronize()
    eo, el = compare_prefill(wl, out.o_prefill.cpu().numpy(), out.lse_prefill.cpu().numpy(), kv_heads=[0, 7],
                             row_range=(0, 64))
    assert eo <= O_TOL and el <= LSE_TOL
    eo, el = compare_decode(wl, out.o_decode.cpu().numpy(), out.lse_decode.cpu().numpy(), requests=[0, 15])
    assert eo <= O_TOL and el <= LSE_TOL
    memo = TunedOptions(reps=3)
    a = memo.options(batch)
    b = memo.options(make_batch(batch.shape, chunk=256, offset=1700, decode_ctx=[2000] * 16))  # same buckets
    assert a is b and len(memo.memo) == 1
