cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( for c in c1 c3_tp8_rank c2_b64; do for m in fused decode; do timeout 300 python tools/graph_vs_eager.py --config $c --mode $m; done; done ) 2>&1
for m in decode fused; do
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg --clock-control none --csv --log-file gpurun_out/ncu_c1_$m.csv timeout 300 python tools/profile_run.py --config c1 --mode $m --iters 3 --precision 2 > /dev/null 2>&1
echo "== $m"; grep -E "pod_|merge" gpurun_out/ncu_c1_$m.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(pod::RunParams.*) Command line profiler metrics//' | tail -8
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "graph or split_invariance or deterministic" 2>&1 | tail -2
