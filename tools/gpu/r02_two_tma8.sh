#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_twolevel.py -x -q 2>&1 | tail -2
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' \
  '[{"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_DIAG": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_NSLOT": 24}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_NSLOT": 32}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_NSLOT": 64}]'
timeout 120 python tools/gpu/two_trace.py
TILEFFT_TWO_DIAG=1 timeout 120 python tools/gpu/two_trace.py
