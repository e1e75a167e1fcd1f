cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_tp.py -q -x -k "split or short or wave or deterministic or graph or full_size_auto or tp_sharded or matches_oracle" > gpurun_out/merge_tests.log 2>&1; echo "rc=$?" >> gpurun_out/merge_tests.log
tail -3 gpurun_out/merge_tests.log; grep -E "^E  |FAILED" gpurun_out/merge_tests.log | head -10
for c in c1 c3_tp8_rank c3_tp4_rank c2_b8 c2_b64; do for m in fused decode; do timeout 300 python tools/graph_vs_eager.py --config $c --mode $m; done; done 2>&1 | cut -c1-150
