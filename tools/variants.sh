#!/bin/bash
# build/variants.sh TAG "EXTRA NVCC FLAGS" -- builds build/lib_TAG.so
set -e
cd "$(dirname "$0")/../paper_2007_00094_b200/csrc"; mkdir -p ../../build
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false $2 \
  -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v -shared -o ../../build/lib_$1.so ef_kernels.cu ef_capi.cu 2> ../../build/ptxas_$1.log
