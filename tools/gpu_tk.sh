cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c2_b16 c2_b32 c2_b64 c3_tp2_rank c3_tp4_rank c3_tp8_rank c4 c1; do echo "== $c"; bash tools/exp.sh $c 2:32:8 2:64:8; done 2>&1
timeout 1200 python tools/sweep.py --chunks 512,2048 --ctx 4096,16384 --batches 8,64 --policy 7 > gpurun_out/tk_sweep_auto.jsonl 2>&1
