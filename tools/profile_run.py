"""Runs one configuration in a given mode for ncu captures / role-log timelines.

  python tools/profile_run.py --config c2_b64 --mode fused --iters 3 [--roles out.json]
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
from bench import CONFIGS  # noqa: E402
from paper_2410_18038_b200.hybrid import PodAttention  # noqa: E402
from paper_2410_18038_b200.workload import build_workload, make_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2_b64")
    ap.add_argument("--mode", default="fused")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--policy", type=int, default=8)
    ap.add_argument("--tile-mode", type=int, default=1)
    ap.add_argument("--decode-splits", type=int, default=0)
    ap.add_argument("--roles", default="")
    ap.add_argument("--precision", type=int, default=0)
    ap.add_argument("--split-wave-cap", type=int, default=0)
    ap.add_argument("--nsm", type=int, default=0, help="plan for this many SMs (the grid)")
    a = ap.parse_args()
    hq, hkv, chunk, off, b, ctx = CONFIGS[a.config]
    b_ = b
    shape = pkg.ModelShape(hq, hkv, 128, math.sqrt(128))
    batch = make_batch(shape, chunk=chunk, offset=off, decode_ctx=[ctx] * b)
    wl = build_workload(batch, device="cuda")
    import dataclasses
    gpu = pkg.GpuSpec.from_device(0)
    if a.nsm:
        gpu = dataclasses.replace(gpu, num_sms=a.nsm)
    op = PodAttention(batch, gpu=gpu, options=pkg.PlanOptions(policy=a.policy, tile_mode=a.tile_mode,
                                                     decode_splits=a.decode_splits, precision=a.precision,
                                                     split_wave_cap=a.split_wave_cap))
    log = op.enable_role_log(768 * 8 + 1024) if a.roles else None
    out = op.alloc_outputs()
    evs = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op.run(wl.q_prefill, wl.q_decode, wl.k_pool, wl.v_pool, wl.page_indptr, wl.page_indices, out=out,
               mode=a.mode)
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    print("event times (us):", [round(x.elapsed_time(y) * 1000, 1) for x, y in evs])
    if log is not None:
        allrec = log.view(-1, 8).cpu()
        nrec = int(op.info.num_prefill_ctas + op.info.num_decode_ctas)
        rec = allrec[:nrec].tolist()
        tr = allrec[nrec:].tolist()
        print("trace words nonzero:", int((allrec[nrec:] != 0).sum()), "policy", a.policy)
        if any(any(x) for x in tr) and op.info.policy == 7:
            print("trace (warpspec): t | A: swait, sok, w0 done, w3 done, mma pA seen, PV_A committed, QK_A committed | B: swait, sok, w0 done, w3 done | mma: vfull ok, PV_A issued, kfull ok, pB seen")
            base = tr[0][0]
            for t in list(range(0, 10)) + list(range(100, 104)):
                row = tr[t][:7] + tr[384 + t][:4] + tr[384 + t][4:8]
                print(t, [((x - base) & 0xffffffff) if x else None for x in row])
        elif any(any(x) for x in tr):
            import os
            print("trace: t | sfull_wait_begin, sfull_ok, softmax_done(pre pv wait), mma_pfull_seen, mma_vfull_ok, mma_kfull_ok(QK t+2), pv_wait_ok, mma_pv_issued | arrive w0..w3, K(t) issue begin/end, V(t) issue begin/end | mma: pv done(probe), qk issued, qk done(probe)")
            base = tr[0][0]
            for t in list(range(0, 12)) + list(range(100, 106)):
                row = tr[t] + tr[256 + t] + tr[512 + t][:3]
                print(t, [((x - base) & 0xffffffff) if x else None for x in row])
        t0 = min(r[5] for r in rec)
        cta = allrec[nrec + 768:].reshape(-1).tolist()[: 2 * 148] if len(tr) >= 768 + 37 else []
        if cta and any(cta):
            st = [cta[2 * i] for i in range(len(cta) // 2) if cta[2 * i]]
            en = [cta[2 * i + 1] for i in range(len(cta) // 2) if cta[2 * i + 1]]
            first_item = min(r[5] for r in rec if r[3] >= 0)
            last_item = max(r[6] for r in rec if r[3] >= 0)
            print(f"CTA entry spread {(max(st) - min(st)) / 1e3:.2f} us; first entry -> first item "
                  f"{(first_item - min(st)) / 1e3:.2f} us; last item end -> last CTA exit {(max(en) - last_item) / 1e3:.2f} us; "
                  f"first entry -> last exit {(max(en) - min(st)) / 1e3:.2f} us")
        rows = [{"sm": r[0], "ticket": r[1], "op": r[2], "id": r[3], "arrival": r[4],
                 "start_us": (r[5] - t0) / 1000.0, "end_us": ((r[6] - t0) % (1 << 31)) / 1000.0} for r in rec]
        Path(a.roles).write_text(json.dumps(rows))
        for opk, name in ((0, "prefill"), (1, "decode")):
            rs = [r for r in rows if r["op"] == opk]
            if rs:
                dur = sorted(r["end_us"] - r["start_us"] for r in rs)
                print(f"{name}: n={len(rs)} start[min,max]=({min(r['start_us'] for r in rs):.1f},"
                      f"{max(r['start_us'] for r in rs):.1f}) end_max={max(r['end_us'] for r in rs):.1f} "
                      f"dur[p10,p50,p90]=({dur[len(dur)//10]:.1f},{dur[len(dur)//2]:.1f},{dur[9*len(dur)//10]:.1f})")
        ds = [r for r in rows if r["op"] == 1]
        ps = [r for r in rows if r["op"] == 0]
        if ps:  # per-SM prefill item durations in claim order
            import collections as _c
            seq = _c.defaultdict(list)
            for r in sorted(ps, key=lambda r: r["start_us"]):
                seq[r["sm"]].append(round(r["end_us"] - r["start_us"], 1))
            k = [v for v in seq.values() if len(v) >= 2]
            if k:
                f, s2 = sorted(v[0] for v in k), sorted(v[1] for v in k)
                print(f"SMs with >= 2 items: {len(k)}; 1st item p50 {f[len(f)//2]} us, 2nd item p50 {s2[len(s2)//2]} us; "
                      f"sample {k[:4]}")
        if ps:  # per-SM prefill busy time and item count
            import collections as _c
            busy, cnt, last = _c.defaultdict(float), _c.Counter(), _c.defaultdict(float)
            for r in ps:
                busy[r["sm"]] += r["end_us"] - r["start_us"]
                cnt[r["sm"]] += 1
                last[r["sm"]] = max(last[r["sm"]], r["end_us"])
            bl, el = sorted(busy.values()), sorted(last.values())
            print(f"prefill per SM: {len(busy)} SMs, items {dict(_c.Counter(cnt.values()))}, busy us "
                  f"p0/p50/p100 = {bl[0]:.1f}/{bl[len(bl)//2]:.1f}/{bl[-1]:.1f}, last end p0/p50/p100 = "
                  f"{el[0]:.1f}/{el[len(el)//2]:.1f}/{el[-1]:.1f}")
        if ds:
            item_bytes = b_ * ctx * hkv * 128 * 4 / len(ds)  # bf16 K + V of one decode item
            rate = sorted(item_bytes / (r["end_us"] - r["start_us"]) / 1e3 for r in ds)
            print(f"decode item {item_bytes/1e6:.2f} MB; per-CTA GB/s p10/p50/p90 = "
                  f"{rate[len(rate)//10]:.1f}/{rate[len(rate)//2]:.1f}/{rate[9*len(rate)//10]:.1f}")
            if ps:
                t_p = max(r["end_us"] for r in ps)
                t_end = max(r["end_us"] for r in rows)
                done_b = sum(item_bytes * max(0.0, min(1.0, (t_p - r["start_us"]) / (r["end_us"] - r["start_us"])))
                             for r in ds if r["start_us"] < t_p)
                print(f"prefill drains at {t_p:.1f} us (end {t_end:.1f}); decode during prefill phase "
                      f"{done_b/1e9:.3f} GB = {done_b/t_p/1e3:.0f} GB/s; after: "
                      f"{(len(ds)*item_bytes-done_b)/1e9:.3f} GB in {t_end-t_p:.1f} us = "
                      f"{(len(ds)*item_bytes-done_b)/max(t_end-t_p,1e-3)/1e3:.0f} GB/s")
        # concurrency per SM
        import collections
        bysm = collections.defaultdict(list)
        for r in rows:
            bysm[r["sm"]].append(r)
        mx = collections.Counter()
        for smv, rs in bysm.items():
            ev = sorted([(r["start_us"], 1) for r in rs] + [(r["end_us"], -1) for r in rs])
            cur = best = 0
            for _, dlt in ev:
                cur += dlt
                best = max(best, cur)
            mx[best] += 1
        print("max concurrent CTAs per SM histogram:", dict(mx))
    import ctypes as C
    from paper_2410_18038_b200._abi import lib
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    st = lib().pod_attn_occupancy(op.plan.handle, C.byref(a), C.byref(b), C.byref(c))
    print("occupancy (fused, prefill, decode):", st, a.value, b.value, c.value)
    print("ok")


if __name__ == "__main__":
    main()
