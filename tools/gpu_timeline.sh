cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in c3_tp8_rank c1 c2_b64; do for m in decode fused; do
  echo "== $cfg $m"; timeout 300 python tools/profile_run.py --config $cfg --mode $m --iters 3 --precision 2 --roles gpurun_out/roles_${cfg}_$m.json | grep -E "event|prefill:|decode:|decode item|drains"
  python tools/decode_timeline.py gpurun_out/roles_${cfg}_$m.json
done; done > gpurun_out/timeline.log 2>&1
cat gpurun_out/timeline.log
