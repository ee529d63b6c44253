#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_twolevel.py tests/test_gpu_bench_plans.py -q -x -k "not 2e30" 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["2d", 4096, 4096], ["2d", 2048, 2048], ["1d", 26]]' '[{}, {"TILEFFT_TWO_1D": 1}]'
done
