cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c2_b8 c2_b16 c1; do echo "== $c"; for i in 1 2; do bash tools/exp.sh $c 2:0; BENCH_NO_PRESLEEP=1 bash tools/exp.sh $c 2:0; done; done
