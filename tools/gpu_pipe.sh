cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -q -x -k "matches_oracle or precision_modes or causality or split_invariance or peaky or random or c2_b16 or c1 or c5" > gpurun_out/pipe_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pipe_tests.log
tail -2 gpurun_out/pipe_tests.log; grep -E "^E  " gpurun_out/pipe_tests.log | head -5
for c in c2_b8 c2_b16 c2_b32 c1; do echo "== $c"; bash tools/exp.sh $c 2::8; POD_LIB=tools/micro/libpod_nopipe.so bash tools/exp.sh $c 2::8; done 2>&1
POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1 timeout 300 python tools/trace64.py --config c2_b8 --mode prefill 2>&1
