cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do bash tools/exp.sh c1 2:64:7::0:1 2:64:7::0:2; done
bash tools/exp.sh c2_b32 2:64:7::0:1 2:64:7::0:2
