#!/bin/bash
# per-launch lists (time + DRAM bytes) for every config, full ncu captures of the top kernels
mkdir -p gpurun_out
B="python bench.py --configs none --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-cufft"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in batched1024 1d_2e20 1d_2e26 2d_8192 1d_2e30; do
  timeout 600 ncu --metrics $M --clock-control none -c 40 --csv --log-file gpurun_out/launches_$c.csv $B --config $c > /dev/null 2>&1
done
P="ncu --set full --clock-control none --import-source on"
timeout 600 $P -k regex:k_rows_tma -s 3 -c 1 -o gpurun_out/prof_rows_tma $B > /dev/null 2>&1
timeout 600 $P -k regex:k_two_tma -s 1 -c 1 -o gpurun_out/prof_two_tma $B --config 2d_8192 > /dev/null 2>&1
timeout 600 $P -k regex:k_comb_tma -s 2 -c 2 -o gpurun_out/prof_comb_2e26 $B --config 1d_2e26 > /dev/null 2>&1
timeout 600 $P -k regex:k_final_t -s 1 -c 1 -o gpurun_out/prof_final_2e26 $B --config 1d_2e26 > /dev/null 2>&1
timeout 900 $P -k regex:k_comb_tma -s 2 -c 1 -o gpurun_out/prof_comb_2e30 $B --config 1d_2e30 > /dev/null 2>&1
ls -la gpurun_out
