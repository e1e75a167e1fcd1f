"""Turn one `tools/gpu_evidence_r2.sh` capture (gpurun_out/ev_*) into the tracked
profiles/<round>/ files: bench lines, per-config lines, the reference arm, ncu
summaries, the launch list, the C5 sweep table, logs.

    python tools/evidence_to_profiles.py [--src gpurun_out] [--dst profiles/round2]
"""
import argparse
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CONFIGS = ["c1", "c2_b8", "c2_b16", "c2_b32", "c2_b64", "c3_tp2_rank", "c3_tp4_rank", "c3_tp8_rank", "c4"]
NCU = {  # report -> (summary file, title)
    "ev_ncu_c2b64_fused": ("ncu_c2b64_fused.md", "c2b64_fused"),
    "ev_ncu_c2b8_prefill": ("ncu_c2b8_prefill.md", "c2b8_prefill"),
    "ev_ncu_c2_prefill_2cta": ("ncu_c2_prefill_2cta.md", "c2_prefill_2cta"),
    "ev_ncu_c2b64_decode": ("ncu_c2b64_decode.md", "c2b64_decode"),
    "ev_ncu_oproj": ("ncu_oproj.md", "oproj"),
}


def last_json(path: Path):
    for line in reversed(path.read_text().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    raise ValueError(f"no JSON line in {path}")


def sweep_md(rows, round1):
    r1 = {(r["chunk"], r["ctx"], r["batch"]): r["fused_us"] for r in round1}
    out = ["# C5 sweep (round 2, final code): prefill chunk x context x decode batch, fused vs serial vs combined "
           "roofline", "",
           "Source: `tools/sweep.py` on one B200 (Llama-3-8B shape 32 Q / 8 KV / d 128, bf16, page 16, AUTO policy, "
           "default POD_PRECISION_F16PV, L2 flushed, median of 5), run by `tools/gpu_evidence_r2.sh`. The last column "
           "is the round-1 fused time of the same point (`profiles/round1/sweep_c5.jsonl`).", "",
           "| chunk | ctx | B | kernel | fused µs | serial µs | prefill µs | decode µs | speedup | fused/max | "
           "roofline µs | % roofline | round 1 fused µs |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    ratios = []
    for r in rows:
        key = (r["chunk"], r["ctx"], r["batch"])
        old = r1.get(key)
        if old:
            ratios.append(old / r["fused_us"])
        out.append(f"| {r['chunk']} | {r['ctx']} | {r['batch']} | {r['policy']} | {r['fused_us']} | {r['serial_us']} | "
                   f"{r['prefill_us']} | {r['decode_us']} | {r['speedup']} | {r['fused_vs_max_alone']} | "
                   f"{r['roofline_us']} | {round(100 * r['roofline_frac'])} % | {old if old else '-'} |")
    sp = [r["speedup"] for r in rows]
    vm = [r["fused_vs_max_alone"] for r in rows]
    geo = 1.0
    for x in ratios:
        geo *= x
    geo = geo ** (1 / len(ratios)) if ratios else float("nan")
    out += ["", f"{len(rows)} points: speedup vs serial {min(sp):.3f}-{max(sp):.3f}x; fused within {max(vm):.3f}x of "
                f"max(alone) everywhere; round-1 -> round-2 fused time ratio {min(ratios):.2f}-{max(ratios):.2f}x "
                f"(geomean {geo:.3f}x)."]
    return "\n".join(out) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default=str(ROOT / "gpurun_out"))
    ap.add_argument("--dst", default=str(ROOT / "profiles" / "round2"))
    a = ap.parse_args()
    src, dst = Path(a.src), Path(a.dst)
    dst.mkdir(parents=True, exist_ok=True)
    # bench lines
    for i, name in ((1, "bench_c2_b64.json"), (2, "bench_c2_b64_run2.json")):
        (dst / name).write_text(json.dumps(last_json(src / f"ev_bench_{i}.json"), indent=1) + "\n")
    (dst / "bench_reference_arm.json").write_text(json.dumps(last_json(src / "ev_bench_ref.json"), indent=1) + "\n")
    with open(dst / "bench_all_configs.jsonl", "w") as f:
        for c in CONFIGS:
            f.write(json.dumps(last_json(src / f"ev_cfg_{c}.json")) + "\n")
    # ncu summaries + the headline kernel's DRAM traffic
    for rep, (md, title) in NCU.items():
        p = src / f"{rep}.ncu-rep"
        if (src / f"{rep}.md").exists():  # summarised on the box (the reports stay there)
            (dst / md).write_text((src / f"{rep}.md").read_text())
        elif p.exists():
            txt = subprocess.run([sys.executable, "tools/ncu_summary.py", str(p.resolve().relative_to(ROOT)),
                                  "--title", title], capture_output=True, text=True, check=True, cwd=ROOT).stdout
            (dst / md).write_text(txt)
    if (src / "ev_launches.md").exists():
        (dst / "launches.md").write_text((src / "ev_launches.md").read_text())
    elif (src / "ev_launches.csv").exists():
        txt = subprocess.run([sys.executable, "tools/ncu_summary.py", "--launches",
                              str((src / "ev_launches.csv").resolve().relative_to(ROOT))], capture_output=True,
                             text=True, check=True, cwd=ROOT).stdout
        (dst / "launches.md").write_text(txt)
    # sweep
    rows = [json.loads(x) for x in (src / "ev_sweep_c5.jsonl").read_text().splitlines() if x.startswith("{")]
    (dst / "sweep_c5.jsonl").write_text("".join(json.dumps(r) + "\n" for r in rows))
    r1p = ROOT / "profiles" / "round1" / "sweep_c5.jsonl"
    r1 = [json.loads(x) for x in r1p.read_text().splitlines() if x.startswith("{")] if r1p.exists() else []
    (dst / "sweep_c5.md").write_text(sweep_md(rows, r1))
    # logs
    for s, d in (("ev_gputest.log", "gputest_evidence.log"), ("ev_smoke.log", "smoke.log"),
                 ("ev_verify.log", "verify_300.log"), ("ev_oproj.log", "oproj_bench.txt"),
                 ("ev_roles.log", "roles_ws_c2_b64.log"), ("ev_roles_c2_b64.json", "roles_ws_c2_b64.json"),
                 ("ev_sanitize.log", "sanitize_summary.log")):
        if (src / s).exists():
            shutil.copy(src / s, dst / d)
    for tool in ("memcheck", "synccheck", "racecheck"):
        if (src / f"sanitize_{tool}.log").exists():
            shutil.copy(src / f"sanitize_{tool}.log", dst / f"sanitize_{tool}.log")
    serve = src / "ev_serve.log"
    if serve.exists():
        try:
            (dst / "serve_bench.json").write_text(json.dumps(last_json(serve), indent=1) + "\n")
        except ValueError:
            pass
    print("profiles written to", dst)


if __name__ == "__main__":
    main()
