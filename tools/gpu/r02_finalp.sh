#!/bin/bash
# persistent final pass with register prefetch of the next tile (TILEFFT_FINAL_P): parity, then timing
TILEFFT_FINAL_P=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py -x -q -k "fast or 2e26 or 2e30 or batched" 2>&1 | tail -2
export CASE_TIMEOUT=120 REPS=50
python tools/gpu/two_probe.py '[["1d", 26], ["1d", 24], ["1d", 22], ["1d", 20], ["1d", 30]]' '[{}, {"TILEFFT_FINAL_P": 1}]'
