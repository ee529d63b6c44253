#!/bin/bash
# per-item timeline of the 8192^2 column pass with the current defaults (lag 40, 56 slots), full and data-only
timeout 120 python tools/gpu/two_trace.py
TILEFFT_TWO_DIAG=1 timeout 120 python tools/gpu/two_trace.py
TILEFFT_TWO_D=24 TILEFFT_TWO_NSLOT=48 timeout 120 python tools/gpu/two_trace.py
