#!/bin/bash
# comb passes with the exchange in place in the tile slot (TILEFFT_COMB_IP=1)
TILEFFT_COMB_IP=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py -q -x -k "fast_mode_fp32 or inverse or 2e26" 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=100
for i in 1 2; do
python tools/gpu/two_probe.py '[["1d", 26], ["1d", 24], ["1d", 22]]' '[{}, {"TILEFFT_COMB_IP": 1}]'
done
