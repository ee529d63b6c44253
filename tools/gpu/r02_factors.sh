#!/bin/bash
# pass factorisations with the in-place comb kernel
export CASE_TIMEOUT=90 REPS=100
python tools/gpu/two_probe.py '[["1d", 26]]' '[{}, {"TILEFFT_FAST_FACTORS": "1024,256,256"}, {"TILEFFT_FAST_FACTORS": "256,256,1024"}, {"TILEFFT_FAST_FACTORS": "256,512,512"}, {"TILEFFT_FAST_FACTORS": "512,256,512"}, {"TILEFFT_FAST_FACTORS": "1024,512,128"}, {"TILEFFT_FAST_FACTORS": "1024,1024,64"}]'
python tools/gpu/two_probe.py '[["1d", 24]]' '[{}, {"TILEFFT_FAST_FACTORS": "512,256,128"}, {"TILEFFT_FAST_FACTORS": "1024,128,128"}, {"TILEFFT_FAST_FACTORS": "128,256,512"}, {"TILEFFT_FAST_FACTORS": "1024,1024,16"}]'
python tools/gpu/two_probe.py '[["1d", 28]]' '[{}, {"TILEFFT_FAST_FACTORS": "512,512,1024"}, {"TILEFFT_FAST_FACTORS": "1024,1024,256"}, {"TILEFFT_FAST_FACTORS": "512,1024,512"}]'
python tools/gpu/two_probe.py '[["1d", 22]]' '[{}, {"TILEFFT_FAST_FACTORS": "1024,64,64"}, {"TILEFFT_FAST_FACTORS": "256,256,64"}]'
