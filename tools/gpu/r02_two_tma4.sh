#!/bin/bash
TILEFFT_TWO_KERNEL=1 timeout 300 python -m pytest tests/test_gpu_twolevel.py -x -q 2>&1 | tail -3
python tools/gpu/two_probe.py '[["1d", 26], ["2d", 8192, 8192]]' \
  '[{"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_DIAG": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 16, "TILEFFT_TWO_NSLOT": 20}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 32, "TILEFFT_TWO_NSLOT": 40}]'
REPS=2 timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_two_tma -c 1 -o gpurun_out/two_tma4_full \
  python tools/gpu/two_probe.py --child '["2d", 8192, 8192]' > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/two_tma4_full.ncu-rep > gpurun_out/two_tma4_full.json
