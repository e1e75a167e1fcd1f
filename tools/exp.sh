#!/bin/bash
# Variant sweep for one config: prints the key fields of each bench line.
#   tools/exp.sh CONFIG precision:tile_keys:policy:split_wave_cap:decode_splits ...
cfg=${1:-c2_b64}; shift
for v in "$@"; do
  IFS=: read -r prec tk pol swc ds sb <<< "$v"
  line=$(timeout 300 python bench.py --config $cfg --precision $prec --policy ${pol:-8} --split-wave-cap ${swc:-0} --decode-splits ${ds:-0} --prefill-tile-keys ${tk:-0} --prefill-s-buffers ${sb:-0} --no-cpu-baseline --no-serial-search --steps 10 2>/dev/null | tail -1)
  python - "$v" "$line" <<'PY'
import json,sys
v=sys.argv[1]
try: j=json.loads(sys.argv[2])
except Exception: print(v,"FAILED",sys.argv[2][:200]); sys.exit()
print(f"{v:12s} fused {j['value']:8.1f} serial {j['serial_us']:8.1f} pf {j['prefill_alone_us']:7.1f} dec {j['decode_alone_us']:7.1f} speedup {j['speedup_vs_serial']:.3f} vsmax {j['fused_vs_max_alone']:.3f} roof {j['combined_roofline_frac']:.3f} splits {j['plan']['prefill_splits']}/{j['plan']['decode_splits']} keys {j['plan']['prefill_tile_keys']} mhz {j['clocks'].get('sm_mhz')} {j['clocks'].get('reasons')}")
PY
done
