#!/bin/bash
# 8192-point row kernel at 3 CTAs per SM (register cap 80, spills) vs 2
TILEFFT_ROWS_PF3=1 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twolevel.py -q -x -k "2d or long_rows" 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["2d", 4096, 4096]]' '[{}, {"TILEFFT_ROWS_PF3": 1}]'
done
