cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c2_b64 c4 c3_tp8_rank c2_b32; do echo "== $c"; bash tools/exp.sh $c 2:0:8; POD_LIB=tools/micro/libpod_d5s4.so bash tools/exp.sh $c 2:0:8; done
