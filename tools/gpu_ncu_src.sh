cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pod_sm_kernel -c 1 -o gpurun_out/src_c2b8_prefill python tools/profile_run.py --config c2_b8 --mode prefill --iters 2 --precision 2 > gpurun_out/src1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pod_sm_kernel -c 1 -o gpurun_out/src_c2b64_fused python tools/profile_run.py --config c2_b64 --mode fused --iters 2 --precision 2 > gpurun_out/src2.log 2>&1
ls -la gpurun_out/src_*
