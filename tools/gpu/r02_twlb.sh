#!/bin/bash
# two-level: W_L roots applied in the B items (TILEFFT_TWO_TWLB=1) vs the A items
TILEFFT_TWO_TWLB=1 timeout 600 python -m pytest tests/test_gpu_twolevel.py -x -q -k "2d or schedule or vs_oracle or inverse" 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_TWLB": 1}, {"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_TWLB": 1}]'
done
