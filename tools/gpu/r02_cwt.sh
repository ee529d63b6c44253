#!/bin/bash
TILEFFT_TWO_1D=1 TILEFFT_TWO_CWT=17 timeout 600 python -m pytest tests/test_gpu_twolevel.py -q -x -k "vs_oracle or 2e26 or inverse" 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["1d", 26], ["1d", 24]]' '[{}, {"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_CWT": 17}]'
done
