#!/bin/bash
# two-level: store cache flavours (diag bit 16: plain B output stores instead of .cs; bit 32: plain A scratch
# stores instead of .cg)
TILEFFT_TWO_DIAG=48 timeout 300 python -m pytest tests/test_gpu_twolevel.py -q -x -k "2d_columns" 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192]]' '[{}, {"TILEFFT_TWO_DIAG": 16}, {"TILEFFT_TWO_DIAG": 32}, {"TILEFFT_TWO_DIAG": 48}]'
done
