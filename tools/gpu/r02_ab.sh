#!/bin/bash
# full GPU suite after the cleanup + twiddle placement A/B (same binary, bench timing and ncu)
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.log 2>&1
tools/microbench/twiddle_ab 50 5 > gpurun_out/r02_twiddle_ab_timing.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none \
    -k regex:k_rows_tma --csv --log-file gpurun_out/r02_twiddle_ab_ncu_nocache.csv tools/microbench/twiddle_ab 10 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_rows_tma --csv \
    --log-file gpurun_out/r02_twiddle_ab_ncu_flush.csv tools/microbench/twiddle_ab 10 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_rows_tma -s 2 -c 1 -o gpurun_out/r02_twiddle_ro tools/microbench/twiddle_ab 1 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_rows_tma -s 3 -c 1 -o gpurun_out/r02_twiddle_smem tools/microbench/twiddle_ab 1 1 > /dev/null 2>&1
echo done
