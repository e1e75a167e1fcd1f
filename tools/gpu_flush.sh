cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c1 c3_tp8_rank c2_b8 c2_b64; do for m in fused decode prefill; do timeout 300 python tools/graph_vs_eager.py --config $c --mode $m; done; done
