cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
# conversion cost bound: POD_PRECISION_FAST (bf16 P, no V conversion) vs F16PV (V -> fp16 in smem per tile)
for c in c2_b8 c2_b64; do echo "== $c"; bash tools/exp.sh $c 2:0:3 1:0:3 2:64:7 1:64:7 2:32:7 1:32:7; done
