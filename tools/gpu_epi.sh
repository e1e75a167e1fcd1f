cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for pol in 8 3; do timeout 900 python tools/sweep.py --heads 64,8 --chunks 512,2048 --ctx 4096,16384 --batches 8,64 --policy $pol > gpurun_out/g8_sweep_$pol.jsonl 2>&1; done
python - <<'PY'
import json
rows = {}
for pol in (8, 3):
    for l in open(f"gpurun_out/g8_sweep_{pol}.jsonl"):
        if l.startswith("{") and "fused_us" in l:
            d = json.loads(l); rows.setdefault((d["chunk"], d["ctx"], d["batch"]), {})[pol] = (d["fused_us"], d["policy"], d.get("roofline_frac"))
for k, v in sorted(rows.items()):
    print(k, v)
PY
