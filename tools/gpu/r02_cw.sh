#!/bin/bash
# two-level pass with more compute warps per CTA (register cap 96 / 80)
for cw in 19 23; do
TILEFFT_TWO_CW=$cw timeout 600 python -m pytest tests/test_gpu_twolevel.py -q -x -k "2d or schedule or stress" 2>&1 | tail -1
done
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_CW": 19}, {"TILEFFT_TWO_CW": 23}, {"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_CW": 19}]'
done
