# dev loop: parity subset, variant sweep (POD_LIB builds under tools/micro), 64-key engine trace
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matches_oracle or peaky or causality or split_invariance or precision_modes" > gpurun_out/iter_tests.log 2>&1; echo "rc=$?" >> gpurun_out/iter_tests.log
tail -2 gpurun_out/iter_tests.log
for c in ${CONFIGS:-c2_b8 c2_b16 c2_b32 c2_b64 c1}; do echo "== $c"; bash tools/exp.sh $c 2::8
  for v in $VARIANTS; do echo "-- $v"; POD_LIB=tools/micro/libpod_$v.so bash tools/exp.sh $c 2::8; done; done > gpurun_out/iter_exp.log 2>&1
cat gpurun_out/iter_exp.log
if [ -f tools/micro/libpod_trace.so ]; then
POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1 timeout 300 python tools/trace64.py --config c2_b8 --mode prefill > gpurun_out/iter_trace.log 2>&1
cat gpurun_out/iter_trace.log; fi
