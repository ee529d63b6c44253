#!/bin/bash
# Pass factorisations of 2^26 and 2^28 with the transposed pass-0 -> pass-1 hand-over (the default since it landed)
mkdir -p gpurun_out
F26='[{}, {"TILEFFT_FAST_FACTORS": "256,512,512"}, {"TILEFFT_FAST_FACTORS": "512,256,512"}, {"TILEFFT_FAST_FACTORS": "1024,256,256"}, {"TILEFFT_FAST_FACTORS": "256,256,1024"}, {"TILEFFT_FAST_FACTORS": "1024,512,128"}, {"TILEFFT_FAST_FACTORS": "128,512,1024"}, {"TILEFFT_FAST_FACTORS": "1024,1024,64"}, {"TILEFFT_FAST_FACTORS": "512,1024,128"}]'
for rep in 1 2; do
CASE_TIMEOUT=120 REPS=50 python tools/gpu/two_probe.py '[["1d", 26]]' "$F26"
done
F28='[{}, {"TILEFFT_FAST_FACTORS": "512,512,1024"}, {"TILEFFT_FAST_FACTORS": "512,1024,512"}, {"TILEFFT_FAST_FACTORS": "1024,256,1024"}]'
CASE_TIMEOUT=120 REPS=20 python tools/gpu/two_probe.py '[["1d", 28]]' "$F28"
