cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
POD_LIB=tools/micro/libpod_dual.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_cases.py -x -q 2>&1 | tail -2
for c in c2_b8 c2_b16 c2_b32 c1; do echo "== $c"; bash tools/exp.sh $c 2:64:7::0:2; POD_LIB=tools/micro/libpod_dual.so bash tools/exp.sh $c 2:64:7::0:2; done
