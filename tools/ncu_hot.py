"""Per-instruction view of an ncu source page (SASS) export:
   ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
   python tools/ncu_hot.py src.csv [--min-exec N] [--range a:b]
Prints index, executed count, samples, top stall reasons and the SASS text."""
import csv
import sys

path = sys.argv[1]
min_exec = int(sys.argv[sys.argv.index("--min-exec") + 1]) if "--min-exec" in sys.argv else 0
rng = None
if "--range" in sys.argv:
    a, b = sys.argv[sys.argv.index("--range") + 1].split(":")
    rng = (int(a), int(b))
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows[2:])
print("total samples", tot)
for n, r in enumerate(rows[2:]):
    if rng and not (rng[0] <= n < rng[1]):
        continue
    ex = int(r[ix["Instructions Executed"]] or 0)
    smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    if ex < min_exec and not rng:
        continue
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    sts = " ".join(f"{c}:{v}" for v, c in st if v)
    print(f"{n:5d} {ex:9d} {smp:6d} {100.0*smp/max(tot,1):5.1f}%  {r[ix['Source']].strip()[:70]:70s} {sts}")
