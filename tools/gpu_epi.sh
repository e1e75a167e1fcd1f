cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c2_b32 c2_b64 c3_tp2_rank; do echo "== $c"; bash tools/exp.sh $c 2:32:7 2:64:7::0:1; done
