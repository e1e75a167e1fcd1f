cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2_b8 c2_b16; do echo "== $c"; bash tools/exp.sh $c 2:0:8 2:0:8; done
timeout 900 python tools/fuzz_more.py 300 2>&1 | tail -1
