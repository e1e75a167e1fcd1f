cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/op_bench.log 2>&1; echo "rc=$?" >> gpurun_out/op_bench.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
   bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-serial-search > gpurun_out/op_tp2.log 2>&1; echo "rc=$?" >> gpurun_out/op_tp2.log
tail -2 gpurun_out/op_bench.log | cut -c1-200
python - <<'PY'
import json
for f in ("gpurun_out/op_bench.log", "gpurun_out/op_tp2.log"):
    for l in open(f):
        if l.startswith("{"):
            j = json.loads(l); print(f, j["value"], j.get("oproj"), j.get("tp_check"))
PY
