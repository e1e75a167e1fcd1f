#!/bin/bash
# 128-key pair engine: first parity check, then timings against the 64-key engine
set -x
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "test_matches_oracle and hybrid_gqa4 and fused" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "128 or matches_oracle" 2>&1 | tail -8
for c in c2_b8 c2_b16 c2_b32 c1; do echo "== $c"; bash tools/exp.sh $c 2:64 2:128; done
