# Round-2 evidence capture on one B200 (gpurun from the repo root).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/ev_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_gputest.log
bash tools/sanitize.sh > gpurun_out/ev_sanitize.log 2>&1
for i in 1 2; do timeout 900 python bench.py > gpurun_out/ev_bench_$i.json 2> gpurun_out/ev_bench_$i.err; done
for c in c1 c2_b8 c2_b16 c2_b32 c2_b64 c3_tp2_rank c3_tp4_rank c3_tp8_rank c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-oproj > gpurun_out/ev_cfg_$c.json 2> gpurun_out/ev_cfg_$c.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pod|merge|append|oproj" -c 200 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-serial-search > gpurun_out/ev_b_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pod_sm_kernel -c 1 -o gpurun_out/ev_ncu_c2b64_fused python tools/profile_run.py --config c2_b64 --mode fused --iters 2 --precision 2 > gpurun_out/ev_ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pod_sm_kernel -c 1 -o gpurun_out/ev_ncu_c2b8_prefill python tools/profile_run.py --config c2_b8 --mode prefill --iters 2 --precision 2 > gpurun_out/ev_ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pod_fused_kernel -c 1 -o gpurun_out/ev_ncu_c2_prefill_2cta python tools/profile_run.py --config c2_b8 --mode prefill --policy 3 --iters 2 --precision 2 > gpurun_out/ev_ncu4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pod_sm_kernel -c 1 -o gpurun_out/ev_ncu_c2b64_decode python tools/profile_run.py --config c2_b64 --mode decode --iters 2 --precision 2 > gpurun_out/ev_ncu3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:oproj -c 1 -o gpurun_out/ev_ncu_oproj python tools/oproj_bench.py > gpurun_out/ev_ncu5.log 2>&1
timeout 300 python tools/oproj_bench.py > gpurun_out/ev_oproj.log 2>&1
timeout 200 python tools/profile_run.py --config c2_b64 --mode fused --iters 3 --precision 2 --roles gpurun_out/ev_roles_c2_b64.json > gpurun_out/ev_roles.log 2>&1
timeout 600 python tools/serve_bench.py > gpurun_out/ev_serve.log 2>&1
timeout 600 python -m paper_2410_18038_b200.verify --instances 300 > gpurun_out/ev_verify.log 2>&1; echo "verify rc=$?" >> gpurun_out/ev_verify.log
timeout 1500 python tools/sweep.py > gpurun_out/ev_sweep_c5.jsonl 2> gpurun_out/ev_sweep.err
# summaries on the box (gpurun copies back <= 64 MiB): the .ncu-rep files stay behind
for r in gpurun_out/ev_ncu_*.ncu-rep; do python tools/ncu_summary.py "$r" --title "$(basename "$r" .ncu-rep | sed 's/^ev_ncu_//')" > "${r%.ncu-rep}.md" 2>/dev/null; done
python tools/ncu_summary.py --launches gpurun_out/ev_launches.csv > gpurun_out/ev_launches.md 2>/dev/null
mkdir -p /tmp/ncu_reps && mv gpurun_out/ev_ncu_*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
ls gpurun_out | grep ev_ | wc -l
