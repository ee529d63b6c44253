#!/bin/bash
# comb passes: L1 prefetch of the inter-pass root table lines before the butterflies (TILEFFT_COMB_PFR)
TILEFFT_COMB_PFR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fast_mode_fp32 or fast_mode_fp64 or inverse" 2>&1 | tail -1
export CASE_TIMEOUT=120 REPS=50
for i in 1 2; do
python tools/gpu/two_probe.py '[["1d", 26], ["1d", 24], ["1d", 30]]' '[{}, {"TILEFFT_COMB_PFR": 1}]'
done
