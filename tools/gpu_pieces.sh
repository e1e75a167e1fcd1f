cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "balanced_prefill_pieces" 2>&1 | tail -5
# balanced pieces (AUTO) vs dynamic items: bench.py --prefill-balance
for c in c2_b8 c2_b16 c2_b32 c2_b64 c1 c3_tp8_rank; do echo "== $c"
  for bal in 1 2; do
    line=$(timeout 300 python bench.py --config $c --prefill-balance $bal --no-cpu-baseline --no-serial-search --steps 10 2>/dev/null | tail -1)
    python -c "import json,sys; j=json.loads(sys.argv[1]); print('bal',sys.argv[2],'fused',j['value'],'pf',j['prefill_alone_us'],'dec',j['decode_alone_us'],'roof',j['combined_roofline_frac'],'pieces',j['plan'].get('prefill_balanced'),j['plan']['prefill_ctas'])" "$line" $bal || echo "FAILED $line"
  done
done 2>&1
