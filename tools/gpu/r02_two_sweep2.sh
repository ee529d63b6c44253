#!/bin/bash
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192]]' '[{}, {"TILEFFT_TWO_D": 24, "TILEFFT_TWO_NSLOT": 40}, {"TILEFFT_TWO_D": 32, "TILEFFT_TWO_NSLOT": 48}, {"TILEFFT_TWO_D": 48, "TILEFFT_TWO_NSLOT": 64}, {"TILEFFT_TWO_D": 40, "TILEFFT_TWO_NSLOT": 48}, {"TILEFFT_TWO_D": 40, "TILEFFT_TWO_NSLOT": 72}]'
done
