#!/bin/bash
# 3-pass factor order with the current kernels (transposed hand-over, k_comb_h3, chunk-first final): make_plan order vs ascending
mkdir -p gpurun_out
for rep in 1 2; do
CASE_TIMEOUT=120 REPS=30 python tools/gpu/two_probe.py '[["1d", 26]]' '[{}, {"TILEFFT_FAST_FACTORS": "256,512,512"}, {"TILEFFT_FAST_FACTORS": "512,256,512"}]'
CASE_TIMEOUT=120 REPS=10 python tools/gpu/two_probe.py '[["1d", 28]]' '[{}, {"TILEFFT_FAST_FACTORS": "512,512,1024"}, {"TILEFFT_FAST_FACTORS": "512,1024,512"}]'
CASE_TIMEOUT=120 REPS=30 python tools/gpu/two_probe.py '[["1d", 25]]' '[{}, {"TILEFFT_FAST_FACTORS": "256,256,512"}]'
CASE_TIMEOUT=120 REPS=10 python tools/gpu/two_probe.py '[["1d", 29]]' '[{}, {"TILEFFT_FAST_FACTORS": "512,1024,1024"}]'
done
