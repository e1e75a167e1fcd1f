cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "f16pv or matches_oracle or peaky or causality" > gpurun_out/f16pv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f16pv_tests.log
tail -3 gpurun_out/f16pv_tests.log
for c in c2_b8 c2_b16 c2_b32 c2_b64 c1 c4 c3_tp8_rank; do echo "== $c"; bash tools/exp.sh $c 0::8 2::8; done > gpurun_out/f16pv_exp.log 2>&1
cat gpurun_out/f16pv_exp.log
