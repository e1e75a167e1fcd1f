cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1
for c in c1 c3_tp8_rank c2_b64; do for m in decode fused prefill; do echo "== $c $m"; timeout 300 python tools/profile_run.py --config $c --mode $m --iters 3 --precision 2 --roles gpurun_out/r.json 2>&1 | grep -E "event|CTA entry|prefill:|decode:"; done; done
