#!/bin/bash
# two-level pass: per-item timeline and the data-movement-only ceiling (diag=1) for 8192^2 columns
timeout 120 python tools/gpu/two_trace.py
TILEFFT_TWO_DIAG=1 timeout 120 python tools/gpu/two_trace.py
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' \
  '[{"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_DIAG": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_DIAG": 3}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 12}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 48, "TILEFFT_TWO_NSLOT": 64}]'
