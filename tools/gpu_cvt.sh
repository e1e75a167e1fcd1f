cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "matches_oracle or precision_modes or causality or split_invariance or peaky or random or graph or deterministic" > gpurun_out/cvt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cvt_tests.log
tail -2 gpurun_out/cvt_tests.log; grep -E "^E  " gpurun_out/cvt_tests.log | head -5
for c in c2_b8 c2_b16 c2_b64 c3_tp8_rank c1; do echo "== $c"; bash tools/exp.sh $c 2::8; POD_LIB=tools/micro/libpod_softcvt.so bash tools/exp.sh $c 2::8; done 2>&1
