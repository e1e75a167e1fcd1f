# Round-end evidence capture on one B200 (run via gpurun from the repo root):
# GPU tests, two bench lines, the ncu launch list of a bench run, ncu --set full of the
# warp-specialised kernel (fused / prefill-only / decode-only), the role log and the C5 sweep.
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py > gpurun_out/bench_final_$i.json 2> gpurun_out/bench_final_$i.err; tail -c 400 gpurun_out/bench_final_$i.json; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pod|merge|append" -c 200 --csv --log-file gpurun_out/launches_ws4.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1
for m in fused prefill decode; do timeout 300 ncu --set full --clock-control none --import-source on -k regex:pod_sm_kernel -c 1 -o gpurun_out/ncu_ws_$m python tools/profile_run.py --config c2_b64 --mode $m --policy 7 --iters 2 > gpurun_out/ncu_$m.log 2>&1; done
timeout 200 python tools/profile_run.py --config c2_b64 --mode fused --iters 3 --roles gpurun_out/roles_ws_c2_b64.json > gpurun_out/roles.log 2>&1
timeout 1200 python tools/sweep.py > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep.err
ls -la gpurun_out | tail -20
