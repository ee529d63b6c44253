#!/bin/bash
# two-level loader pre-polls the next item's dependency counter
timeout 900 python -m pytest tests/test_gpu_twolevel.py -x -q 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_1D": 1}]'
done
timeout 120 python tools/gpu/two_trace.py
