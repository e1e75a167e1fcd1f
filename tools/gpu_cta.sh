cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for nsm in 74 128; do echo "== c2_b8 prefill dynamic nsm $nsm"; timeout 300 python tools/profile_run.py --config c2_b8 --mode prefill --iters 3 --precision 2 --roles gpurun_out/r.json --nsm $nsm 2>&1 | grep -E "event|prefill|SMs with"; done
