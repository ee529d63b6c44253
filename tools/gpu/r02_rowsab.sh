#!/bin/bash
# Headline kernel load-path A/B (tools/microbench/rows_ab.cu): TMA ring vs direct LDG variants.
set -e
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr \
  -o gpurun_out/rows_ab tools/microbench/rows_ab.cu
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > gpurun_out/rows_ab_clocks.txt
timeout 300 gpurun_out/rows_ab 50 5 2>&1 | tee gpurun_out/rows_ab.txt
timeout 300 gpurun_out/rows_ab 50 5 2>&1 | tee -a gpurun_out/rows_ab.txt
