cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c2_b8 c2_b16; do
  for l in poly2 poly3 k2v2d2 k2v2d2p2; do echo "== $c $l"; POD_LIB=tools/micro/libpod_$l.so bash tools/exp.sh $c 2:64 2:128; done
done 2>&1
