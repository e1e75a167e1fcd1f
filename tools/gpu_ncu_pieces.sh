cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for bal in 1 2; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/ncu_pieces_$bal.csv -k regex:pod_sm_kernel timeout 300 python tools/profile_run.py --config c2_b8 --mode prefill --iters 2 --precision 2 --prefill-balance $bal > /dev/null 2>&1
echo "== balance $bal"; grep -E "pod_sm" gpurun_out/ncu_pieces_$bal.csv | awk -F'","' '{print $(NF-3), $(NF-2), $NF}' | tail -10
done
