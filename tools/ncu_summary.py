"""Summarise ncu captures into markdown for profiles/.

  python tools/ncu_summary.py report.ncu-rep [--title T] > profiles/roundN/x.md
  python tools/ncu_summary.py --launches launches.csv > profiles/roundN/launches.md
"""
import argparse
import collections
import csv
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep, title):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units = rows[0], rows[1]
    print(f"# {title}\n\nSource: `{rep}` (ncu --set full --clock-control none; one replayed launch per row).\n")
    cols = [(hdr.index(m), name, units[hdr.index(m)]) for m, name in METRICS if m in hdr]
    kname = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
    for r in rows[2:]:
        if kname is not None:
            print(f"## {r[kname][:120]}\n")
        print("| metric | value |\n|---|---|")
        for i, name, u in cols:
            print(f"| {name} | {r[i]} {u} |")
        print()
    sass = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    if len(sass) > 2:
        h = sass[1]
        data = []
        for x in sass[2:]:
            if x and x[0] == "Kernel Name":
                break  # first kernel only
            if len(x) == len(h):
                data.append(x)
        iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        tot_e = sum(int(x[iE] or 0) for x in data) or 1
        tot_w = sum(int(x[iW] or 0) for x in data) or 1
        ops_e, ops_w = collections.Counter(), collections.Counter()
        for x in data:
            m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", x[iS])
            op = m.group(2) if m else "?"
            ops_e[op] += int(x[iE] or 0)
            ops_w[op] += int(x[iW] or 0)
        print("## SASS instruction mix (first kernel in the report)\n\n| opcode | executed % | stall samples % |\n|---|---|---|")
        for op, v in ops_e.most_common(16):
            print(f"| {op} | {100 * v / tot_e:.1f} | {100 * ops_w[op] / tot_w:.1f} |")
        print("\n## Top stall sites\n\n| samples % | executed | instruction |\n|---|---|---|")
        for x in sorted(data, key=lambda x: -int(x[iW] or 0))[:12]:
            print(f"| {100 * int(x[iW]) / tot_w:.1f} | {x[iE]} | `{x[iS].strip()[:80]}` |")
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    iK, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    print(f"# Launch list\n\nSource: `{path}` (`ncu --metrics gpu__time_duration.sum --clock-control none`, cold-cache, "
          f"serialised: compare shares, not absolutes).\n")
    print("| # | kernel | duration (us) |\n|---|---|---|")
    n = 0
    for r in rows[start + 1:]:
        if len(r) != len(hdr) or r[iM] != "gpu__time_duration.sum" or not re.search(
                r"pod::|pod_sm_kernel|pod_fused_kernel|merge_kernel|append_kv_kernel", r[iK]):
            continue
        n += 1
        print(f"| {n} | {r[iK][:70]} | {float(r[iV].replace(',', '')) / 1000:.1f} |")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.launches:
        launches(a.launches)
    else:
        summarize(a.report, a.title)
