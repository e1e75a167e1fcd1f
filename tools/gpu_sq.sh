cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "matches_oracle or sq" > gpurun_out/sq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sq_tests.log
tail -3 gpurun_out/sq_tests.log; grep -E "^E  " gpurun_out/sq_tests.log | head -5
for c in c2_b8 c2_b16 c2_b32 c2_b64 c1 c4; do echo "== $c"; bash tools/exp.sh $c 2::8:0:0:1 2::8:0:0:2; done > gpurun_out/sq_exp.log 2>&1
cat gpurun_out/sq_exp.log
