cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1
( timeout 300 python tools/trace64.py --config c2_b8 --mode prefill --engine 3
  timeout 300 python tools/trace64.py --config c2_b8 --mode prefill --engine 3 --chunk 32 ) > gpurun_out/trace64.log 2>&1
cat gpurun_out/trace64.log
