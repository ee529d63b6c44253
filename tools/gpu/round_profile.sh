# Round-end evidence: bench lines for every config, per-launch lists, ncu --set full of the top kernels.
set -x
for c in batched1024 1d_2e20 1d_2e26 2d_8192 1d_2e30; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 --steps 50 2>&1 | tail -1 > gpurun_out/bench_$c.json
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in batched1024 1d_2e20 1d_2e26 2d_8192 1d_2e30; do
  timeout 600 ncu --metrics $M --clock-control none -c 12 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_two -c 1 -o gpurun_out/prof_two_2d \
  python bench.py --config 2d_8192 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows_tma -s 3 -c 1 -o gpurun_out/prof_rows_tma \
  python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_two_2d.ncu-rep gpurun_out/prof_rows_tma.ncu-rep > gpurun_out/ncu_round.json
