#!/bin/bash
# two-level kernel after the s_cnt fix: parity tests, then repeated runs of default and tuned lag/slot settings
timeout 600 python -m pytest tests/test_gpu_twolevel.py tests/test_gpu_bench_plans.py -x -q 2>&1 | tail -2
export CASE_TIMEOUT=60 REPS=300
for i in 1 2 3 4 5; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' \
  '[{}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 40, "TILEFFT_TWO_NSLOT": 56}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 32, "TILEFFT_TWO_NSLOT": 48}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 80, "TILEFFT_TWO_NSLOT": 96}]'
done
