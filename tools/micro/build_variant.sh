#!/bin/bash
# Experiment build of the product library with extra -D flags:
#   tools/micro/build_variant.sh NAME -DPOD_X=1 ...  ->  tools/micro/libpod_NAME.so
# (select at run time with POD_LIB=tools/micro/libpod_NAME.so)
set -e
name=$1; shift
cd "$(dirname "$0")/../.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -O3 --expt-relaxed-constexpr "$@" -shared -o tools/micro/libpod_$name.so \
  paper_2410_18038_b200/csrc/pod_attn.cu paper_2410_18038_b200/csrc/pod_plan.cpp
