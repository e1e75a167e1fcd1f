cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1
( true
  for k in 64 128; do timeout 300 python tools/trace64.py --config c2_b8 --mode prefill --keys $k --chunk 64; done ) > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
