cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_cases.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
for c in c2_b8 c2_b16; do echo "== $c"; bash tools/exp.sh $c 2:0:8 2:0:8 ; done
