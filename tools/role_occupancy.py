#!/usr/bin/env python3
"""Per-role SM occupancy from a role log (tools/profile_run.py --roles X.json):
fraction of SM-time (over the launch span) in which a prefill item, a decode item,
or both are resident on the SM -- the "SM occupancy split per role" evidence.

  python tools/role_occupancy.py roles.json
"""
import json
import sys

import numpy as np


def main():
    rows = json.load(open(sys.argv[1]))
    t_end = max(r["end_us"] for r in rows)
    grid = np.linspace(0.0, t_end, 2001)
    by_sm = {}
    for r in rows:
        by_sm.setdefault(r["sm"], []).append(r)
    pf = np.zeros((len(by_sm), grid.size), bool)
    dc = np.zeros_like(pf)
    for i, (sm, rs) in enumerate(sorted(by_sm.items())):
        for r in rs:
            m = (grid >= r["start_us"]) & (grid < r["end_us"])
            (pf if r["op"] == 0 else dc)[i] |= m
    both = pf & dc
    out = {"span_us": round(t_end, 1), "sms": len(by_sm),
           "prefill_resident_frac": round(float(pf.mean()), 3), "decode_resident_frac": round(float(dc.mean()), 3),
           "both_resident_frac": round(float(both.mean()), 3),
           "idle_frac": round(float((~pf & ~dc).mean()), 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
