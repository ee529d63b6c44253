#!/bin/bash
# small (L2-resident) multi-pass plans: 4-comb/4-row tiles (default) vs the TMA in-place comb / persistent final
for v in 1 2 3; do TILEFFT_NO_SMALL=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fast_mode_fp32 or inverse" 2>&1 | tail -1; done
export CASE_TIMEOUT=60 REPS=500
for i in 1 2; do
python tools/gpu/two_probe.py '[["1d", 14], ["1d", 16], ["1d", 18], ["1d", 20], ["1d", 22]]' '[{}, {"TILEFFT_NO_SMALL": 1}, {"TILEFFT_NO_SMALL": 2}, {"TILEFFT_NO_SMALL": 3}]'
done
