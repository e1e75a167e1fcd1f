cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export POD_TRACE=1
( for v in trace trspinm trspinb; do echo "-- $v"; POD_LIB=tools/micro/libpod_$v.so timeout 300 python tools/trace64.py --config c2_b8 --mode prefill; done ) > gpurun_out/trace64.log 2>&1
unset POD_TRACE
( for c in c2_b8 c2_b16; do echo "== $c"; bash tools/exp.sh $c 2::8; for v in spinm spinb; do echo "-- $v"; POD_LIB=tools/micro/libpod_$v.so bash tools/exp.sh $c 2::8; done; done ) >> gpurun_out/trace64.log 2>&1
cat gpurun_out/trace64.log
