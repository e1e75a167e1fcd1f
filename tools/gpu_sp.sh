cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "sp or matches_oracle or random" > gpurun_out/sp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sp_tests.log
tail -2 gpurun_out/sp_tests.log; grep -E "^E  " gpurun_out/sp_tests.log | head -8
for c in c2_b8 c2_b16 c2_b32 c2_b64 c1 c3_tp8_rank; do echo "== $c"; bash tools/exp.sh $c 2::8 2::8:0:0:3; done 2>&1
