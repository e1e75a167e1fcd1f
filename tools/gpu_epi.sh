cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
for c in c1 c2_b8 c2_b64 c3_tp8_rank c4; do echo "== $c"; bash tools/exp.sh $c 2:0; done
POD_LIB=tools/micro/libpod_trace.so POD_TRACE=1 timeout 300 python tools/trace64.py --config c1 --mode prefill --keys 64 --raw | tail -3
