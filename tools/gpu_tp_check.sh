#!/bin/bash
# GPU-box check of the bench paths added for the TP / serial / CPU-baseline work.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tp.py -q -rf > gpurun_out/gputest_tp.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_tp.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-serial-search > gpurun_out/bench_tp2_gloo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_tp2_gloo.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
nproc >> gpurun_out/bench_ref.log
tail -3 gpurun_out/gputest_tp.log
