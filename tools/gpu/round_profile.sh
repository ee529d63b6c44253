# Round-end evidence: parity suite, bench lines for every config, per-launch lists,
# ncu --set full summaries of the top kernels (reports deleted after summarising,
# so gpurun_out stays under the 64 MiB copy-back limit).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for c in batched1024 1d_2e20 1d_2e26 2d_8192 1d_2e30; do
  timeout 600 python bench.py --config $c --e2e-steps 2 --steps 50 $([ $c != batched1024 ] && echo --no-cpu-baseline) 2>&1 | tail -1 > gpurun_out/bench_$c.json
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in batched1024 1d_2e20 1d_2e26 2d_8192 1d_2e30; do
  timeout 600 ncu --metrics $M --clock-control none -c 12 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
done
P="ncu --set full --clock-control none --import-source on"
timeout 900 $P -k regex:k_two_ws -c 1 -o gpurun_out/prof_two_ws python bench.py --config 2d_8192 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $P -k regex:k_rows_tma -s 3 -c 1 -o gpurun_out/prof_rows_tma python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $P -k regex:k_rows_pf -c 1 -o gpurun_out/prof_rows_pf python bench.py --config 2d_8192 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $P -k regex:k_comb_tma -c 1 -o gpurun_out/prof_comb_2e26 python bench.py --config 1d_2e26 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_two_ws.ncu-rep gpurun_out/prof_rows_tma.ncu-rep gpurun_out/prof_comb_2e26.ncu-rep gpurun_out/prof_rows_pf.ncu-rep > gpurun_out/ncu_round.json
for r in two_ws rows_tma comb_2e26 rows_pf; do
  ncu -i gpurun_out/prof_$r.ncu-rep --page source --csv > gpurun_out/prof_${r}_source.csv 2>&1
  rm -f gpurun_out/prof_$r.ncu-rep
done
