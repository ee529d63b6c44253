#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_twolevel.py -x -q 2>&1 | tail -2
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' \
  '[{"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 32, "TILEFFT_TWO_NSLOT": 48}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 40, "TILEFFT_TWO_NSLOT": 56}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 32, "TILEFFT_TWO_NSLOT": 40}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 48, "TILEFFT_TWO_NSLOT": 64}]'
TILEFFT_TWO_D=40 TILEFFT_TWO_NSLOT=56 timeout 120 python tools/gpu/two_trace.py
