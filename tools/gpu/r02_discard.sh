#!/bin/bash
# k_two_tma: discard consumed scratch lines (default) vs not; DRAM bytes of the column pass for both
timeout 600 python -m pytest tests/test_gpu_twolevel.py -x -q 2>&1 | tail -1
export CASE_TIMEOUT=60 REPS=200
for i in 1 2; do
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_DISCARD": 0}, {"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_DISCARD": 0}]'
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
B="python bench.py --configs none --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-cufft --config 2d_8192"
timeout 300 ncu --metrics $M --clock-control none -k regex:k_two -c 4 --csv --log-file gpurun_out/launches_two_discard1.csv $B > /dev/null 2>&1
TILEFFT_TWO_DISCARD=0 timeout 300 ncu --metrics $M --clock-control none -k regex:k_two -c 4 --csv --log-file gpurun_out/launches_two_discard0.csv $B > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_two_discard1.csv; python tools/launch_table.py gpurun_out/launches_two_discard0.csv
