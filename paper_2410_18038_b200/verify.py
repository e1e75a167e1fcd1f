"""attn-verify on the GPU: the reference CLI's self-check suite (attnsim_cli.cpp:92-190)
run through pod_attn_run on sm_100a.

    python -m paper_2410_18038_b200.verify [--instances 40] [--split-instances 20]
        [--causality-instances 20] [--max-m 256] [--max-n 2048] [--seed 7]
        [--tolerance 2e-3] [--inject-mask-off-by-one]

Suites (same names and output table as the reference; exit 0 = all PASS, 1 = a suite
failed, 2 = configuration / device error, as attnsim_cli.cpp:454-460):

* oracle-equivalence -- random hybrid batches (1-2 KV heads, GQA group 1/2/4, random chunk,
  offset, decode contexts and kernel policy) against a dense float64 softmax(QK^T/scale)V of
  the same bf16 inputs gathered from the paged pool by torch indexing.  The reference
  compares double against long double per element (:66-90); bf16 inputs and fp32
  accumulation make that meaningless here, so the error is max|O - O_ref| / max|O_ref| per
  batch, with the north star's 2e-3 bar; LSE is checked absolutely.
* split-invariance -- decode-only batches, KV splits 2..8 merged vs 1 split (:122-146).
* causality -- perturbing keys after a probe row (+3 on K, -2 on V) leaves the row bit-identical
  (:148-180).  --inject-mask-off-by-one perturbs the row's own last visible key instead, the
  same one-key widening the reference injects, and must FAIL.

The checker is plain PyTorch on the device, not the product path.  Head dim is 128 (the only
head dim the sm_100a kernels build; the reference draws d from the config's list).
"""
from __future__ import annotations

import argparse
import math
import sys
from dataclasses import dataclass

import torch


@dataclass
class SuiteResult:
    name: str
    cases: int = 0
    worst: float = 0.0
    passed: bool = True


def _gather(wl, req: int) -> tuple:
    """K, V of request `req` as [ctx][Hkv][d] float64, gathered through the block table."""
    ps = wl.batch.page_size
    ctx = wl.kv_lens[req]
    a, b = int(wl.page_indptr[req]), int(wl.page_indptr[req + 1])
    pages = wl.page_indices[a:b].long()
    k = wl.k_pool[pages].permute(0, 2, 1, 3).reshape(-1, wl.k_pool.shape[1], wl.k_pool.shape[3])[:ctx]
    v = wl.v_pool[pages].permute(0, 2, 1, 3).reshape(-1, wl.v_pool.shape[1], wl.v_pool.shape[3])[:ctx]
    return k.double(), v.double()


def _dense(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: float, first_visible_limit: torch.Tensor):
    """q [m][Hq][d], k/v [ctx][Hkv][d] float64; row r sees keys j <= limit[r]."""
    g = q.shape[1] // k.shape[1]
    kx, vx = k.repeat_interleave(g, dim=1), v.repeat_interleave(g, dim=1)
    s = torch.einsum("rhd,jhd->hrj", q, kx) / scale
    j = torch.arange(k.shape[0], device=q.device)
    s = s.masked_fill(j[None, None, :] > first_visible_limit[None, :, None], float("-inf"))
    lse = torch.logsumexp(s, dim=-1)                      # [Hq][m]
    o = torch.einsum("hrj,jhd->rhd", torch.softmax(s, dim=-1), vx)
    return o, lse.transpose(0, 1)


def dense_reference(wl) -> dict:
    b = wl.batch
    scale = b.shape.scale
    out = {}
    req = 0
    if b.prefill is not None:
        k, v = _gather(wl, 0)
        m, off = b.prefill.chunk_size, b.prefill.position_offset
        lim = off + torch.arange(m, device=k.device)
        out["o_prefill"], out["lse_prefill"] = _dense(wl.q_prefill.double(), k, v, scale, lim)
        req = 1
    if b.decodes:
        os_, ls_ = [], []
        for i in range(len(b.decodes)):
            k, v = _gather(wl, req + i)
            lim = torch.tensor([k.shape[0] - 1], device=k.device)
            o, lse = _dense(wl.q_decode[i:i + 1].double(), k, v, scale, lim)
            os_.append(o)
            ls_.append(lse)
        out["o_decode"], out["lse_decode"] = torch.cat(os_), torch.cat(ls_)
    return out


def _scale_err(got: torch.Tensor, ref: torch.Tensor) -> float:
    return ((got.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


def _policies():
    from . import _abi
    return [_abi.POD_POLICY_AUTO, _abi.POD_POLICY_COMPLEMENT, _abi.POD_POLICY_WARPSPEC]


def run_suites(a, device="cuda") -> list:
    from .hybrid import PodAttention
    from .pod import ModelShape, PlanOptions
    from .workload import Rng, build_workload, make_batch

    rng = Rng(a.seed)
    d = 128
    suites = []

    s = SuiteResult("oracle-equivalence")
    for i in range(a.instances):
        hkv = rng.next_long(1, 2)
        hq = hkv * [1, 2, 4][rng.next_long(0, 2)]
        shape = ModelShape(hq, hkv, d, math.sqrt(d))
        m = rng.next_long(0, a.max_m)                      # 0 = decode-only batch
        off = rng.next_long(0, max(0, a.max_n - max(m, 1)))
        nd = rng.next_long(0 if m else 1, 4)
        ctxs = [rng.next_long(1, a.max_n) for _ in range(nd)]
        policy = _policies()[rng.next_long(0, 2)]
        batch = make_batch(shape, chunk=m, offset=off, decode_ctx=ctxs)
        wl = build_workload(batch, device=device, seed_q=1000 + i, seed_kv=2000 + i, seed_pages=3000 + i)
        op = PodAttention(batch, options=PlanOptions(policy=policy))
        got = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)
        ref = dense_reference(wl)
        for key in ("o_prefill", "o_decode"):
            if key in ref:
                s.worst = max(s.worst, _scale_err(getattr(got, key), ref[key]))
                lkey = key.replace("o_", "lse_")
                lerr = (getattr(got, lkey).double() - ref[lkey]).abs().max().item()
                if lerr > a.tolerance:
                    s.passed = False
        s.cases += 1
    s.passed = s.passed and s.worst <= a.tolerance
    suites.append(s)

    s = SuiteResult("split-invariance")
    for i in range(a.split_instances):
        hkv = rng.next_long(1, 2)
        shape = ModelShape(hkv * 2, hkv, d, math.sqrt(d))
        batch = make_batch(shape, decode_ctx=[rng.next_long(8, 512)])
        wl = build_workload(batch, device=device, seed_q=4000 + i, seed_kv=5000 + i, seed_pages=6000 + i)
        base = None
        for splits in range(1, 9):
            op = PodAttention(batch, options=PlanOptions(decode_splits=splits))
            o = op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices).o_decode
            if base is None:
                base = o.double()
            else:
                s.worst = max(s.worst, _scale_err(o, base))
        s.cases += 1
    s.passed = s.worst <= a.tolerance
    suites.append(s)

    s = SuiteResult("causality")
    exact = True
    for i in range(a.causality_instances):
        shape = ModelShape(2, 1, d, math.sqrt(d))
        m = rng.next_long(2, 12)
        off = rng.next_long(0, 64)
        batch = make_batch(shape, chunk=m, offset=off)
        wl = build_workload(batch, device=device, seed_q=7000 + i, seed_kv=8000 + i, seed_pages=9000 + i)
        probe = rng.next_long(0, m - 1)
        op = PodAttention(batch, options=PlanOptions(policy=_policies()[i % 3]))
        before = op.run(wl.q_prefill, None, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)
        first = off + probe + (0 if a.inject_mask_off_by_one else 1)
        ps = batch.page_size
        pages = wl.page_indices[int(wl.page_indptr[0]):int(wl.page_indptr[1])].long()
        for j in range(first, off + m):
            pg, slot = int(pages[j // ps]), j % ps
            wl.k_pool[pg, :, slot] = (wl.k_pool[pg, :, slot].float() + 3.0).to(wl.k_pool.dtype)
            wl.v_pool[pg, :, slot] = (wl.v_pool[pg, :, slot].float() - 2.0).to(wl.v_pool.dtype)
        after = op.run(wl.q_prefill, None, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices)
        if not torch.equal(before.o_prefill[probe], after.o_prefill[probe]):
            exact = False
        s.cases += 1
    s.passed = exact
    s.worst = 0.0 if exact else 1.0
    suites.append(s)
    return suites


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="attn-verify", description=__doc__.split("\n\n")[0])
    ap.add_argument("--instances", type=int, default=40)
    ap.add_argument("--split-instances", type=int, default=20)
    ap.add_argument("--causality-instances", type=int, default=20)
    ap.add_argument("--max-m", type=int, default=256)
    ap.add_argument("--max-n", type=int, default=2048)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--tolerance", type=float, default=2e-3)
    ap.add_argument("--inject-mask-off-by-one", action="store_true")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    if a.instances < 0 or a.split_instances < 0 or a.causality_instances < 0 or a.max_m < 1 or a.max_n < 2 \
            or not a.tolerance > 0:
        print("attn-verify: invalid configuration", file=sys.stderr)
        return 2
    if not torch.cuda.is_available():
        print("attn-verify: needs a CUDA device (the suite runs the sm_100a kernels)", file=sys.stderr)
        return 2
    try:
        suites = run_suites(a)
    except Exception as e:  # plan / run errors are configuration errors (exit 2), as in the reference
        print(f"attn-verify: {e}", file=sys.stderr)
        return 2
    print(f"{'suite':<20s} {'cases':>8s} {'max_err':>12s} {'status':>6s}")
    ok = True
    for s in suites:
        print(f"{s.name:<20s} {s.cases:>8d} {s.worst:>12.3e} {'PASS' if s.passed else 'FAIL':>6s}")
        ok = ok and s.passed
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
