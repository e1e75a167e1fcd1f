cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do for c in c2_b16 c1; do echo "== $c"; bash tools/exp.sh $c 2:64:7::0:1 2:64:7::0:2; done; done
