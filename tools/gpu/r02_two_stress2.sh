#!/bin/bash
# reproduce the two-level timeout with the per-CTA watchdog snapshot; 32-row final-pass experiment
export CASE_TIMEOUT=60 REPS=300
REPS=100 python tools/gpu/two_probe.py '[["1d", 26], ["1d", 24], ["1d", 22]]' '[{}, {"TILEFFT_FINAL_F32": 1}]'
for i in 1 2 3 4 5 6; do
python tools/gpu/two_probe.py '[["1d", 26]]' '[{"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 40, "TILEFFT_TWO_NSLOT": 56}, {"TILEFFT_TWO_1D": 1}]'
python tools/gpu/two_probe.py '[["2d", 8192, 8192]]' '[{}]'
done
