#!/bin/bash
# new barrier-free two-level kernel (k_two_tma): parity then timing vs k_two_ws
for K in 2 1; do
  echo "== TILEFFT_TWO_KERNEL=$K tests"
  TILEFFT_TWO_KERNEL=$K timeout 300 python -m pytest tests/test_gpu_twolevel.py -x -q 2>&1 | tail -4
done
CASES='[["1d", 26], ["2d", 8192, 8192], ["2d", 4096, 4096], ["2d", 2048, 2048]]' timeout 300 python tools/gpu/time_cfg.py \
  '[{"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 0}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 2}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_KERNEL": 1}]'
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_two --csv \
  env TILEFFT_TWO_1D=1 TILEFFT_TWO_KERNEL=2 CASES='[["1d", 26], ["2d", 8192, 8192]]' python tools/gpu/time_cfg.py > gpurun_out/two_tma_ncu.csv 2>&1
tail -5 gpurun_out/two_tma_ncu.csv
