#!/bin/bash
# two-level: loader-decoded item geometry (new .so) vs per-unit divisions (libtilefft_b200_prev.so), same box
timeout 600 python -m pytest tests/test_gpu_twolevel.py -q -x 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=300
L=paper_1707_07263_b200/libtilefft_b200.so
cp $L /tmp/new.so
for i in 1 2 3; do
  cp /tmp/new.so $L; echo new; python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_1D": 1}]'
  cp paper_1707_07263_b200/libtilefft_b200_prev.so $L; echo prev; python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_1D": 1}]'
done
cp /tmp/new.so $L
