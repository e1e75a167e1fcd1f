cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2 3 4; do bash tools/exp.sh c1 2:0; done
POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1 timeout 300 python tools/trace64.py --config c1 --mode prefill --keys 64 --raw | head -4
timeout 300 python tools/graph_vs_eager.py --config c1 --mode fused
