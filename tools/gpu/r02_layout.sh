#!/bin/bash
# 2^30 comb-pass layout probe (tools/microbench/comb_layout.cu): read and write row strides varied independently
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gpurun_out/comb_layout tools/microbench/comb_layout.cu
timeout 300 gpurun_out/comb_layout 2>&1 | tee gpurun_out/comb_layout.txt
