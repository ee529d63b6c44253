#!/bin/bash
# 2^30 comb-pass stride probe (tools/microbench/comb_stride.cu): TMA comb-tile copy at pass-0 vs pass-1 strides
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gpurun_out/comb_stride tools/microbench/comb_stride.cu
timeout 300 gpurun_out/comb_stride 30 2>&1 | tee gpurun_out/comb_stride.txt
