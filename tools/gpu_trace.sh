cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1
( for m in prefill; do timeout 300 python tools/trace64.py --config c1 --mode $m --keys 64 --raw; done
  true ) > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
