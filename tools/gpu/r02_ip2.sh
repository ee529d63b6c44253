#!/bin/bash
# in-place comb exchange as the default for L <= 512: full GPU suite; L = 1024 (2^30) variant timing
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
export CASE_TIMEOUT=120 REPS=20
python tools/gpu/two_probe.py '[["1d", 30], ["1d", 28], ["1d", 26], ["1d", 20]]' '[{}, {"TILEFFT_COMB_IP": 1}]'
REPS=200 python tools/gpu/two_probe.py '[["1d", 26], ["1d", 24], ["1d", 22], ["1d", 20], ["1d", 18], ["2d", 8192, 8192], ["2d", 1024, 1024]]' '[{}]'
