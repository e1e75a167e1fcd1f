"""Decode-item timeline summary from a role log (tools/profile_run.py --roles X.json):
per-SM item count, busy span, the launch makespan vs the mean per-SM finish time
(imbalance), item duration percentiles and per-item start latency.

  python tools/decode_timeline.py roles.json [item_MB]
"""
import collections
import json
import sys


def main():
    rows = json.load(open(sys.argv[1]))
    item_mb = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    ds = [r for r in rows if r["op"] == 1]
    ps = [r for r in rows if r["op"] == 0]
    t_end = max(r["end_us"] for r in rows)
    by = collections.defaultdict(list)
    for r in ds:
        by[r["sm"]].append(r)
    fin = sorted(max(r["end_us"] for r in rs) for rs in by.values())
    cnt = collections.Counter(len(rs) for rs in by.values())
    dur = sorted(r["end_us"] - r["start_us"] for r in ds)
    first = sorted(min(r["start_us"] for r in rs) for rs in by.values())
    gaps = []
    for rs in by.values():
        rs = sorted(rs, key=lambda r: r["start_us"])
        gaps += [b["start_us"] - a["end_us"] for a, b in zip(rs, rs[1:])]
    gaps.sort()
    q = lambda xs, f: xs[min(len(xs) - 1, int(f * len(xs)))] if xs else float("nan")  # noqa: E731
    print(f"span {t_end:.1f} us; decode items {len(ds)} on {len(by)} SMs, items/SM {dict(cnt)}; prefill items {len(ps)}")
    print(f"SM decode finish: min {fin[0]:.1f} p50 {q(fin, .5):.1f} max {fin[-1]:.1f} (mean {sum(fin)/len(fin):.1f})")
    print(f"first decode start per SM: p50 {q(first, .5):.2f} max {first[-1]:.2f} us")
    print(f"item duration p10/p50/p90/max: {q(dur, .1):.1f}/{q(dur, .5):.1f}/{q(dur, .9):.1f}/{dur[-1]:.1f} us")
    print(f"gap between an SM's consecutive items p50/p90: {q(gaps, .5):.2f}/{q(gaps, .9):.2f} us")
    if item_mb:
        print(f"per-item GB/s p10/p50/p90: {item_mb*1e3/q(dur, .9):.0f}/{item_mb*1e3/q(dur, .5):.0f}/{item_mb*1e3/q(dur, .1):.0f}")


if __name__ == "__main__":
    main()
