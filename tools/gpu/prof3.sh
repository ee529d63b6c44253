# ncu --set full: comb pass (2^30), final pass (2^30), 8192-point rows (2D)
P="ncu --set full --clock-control none --import-source on"
timeout 900 $P -k regex:k_comb_tma -c 1 -o gpurun_out/prof_comb30 python bench.py --config 1d_2e30 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $P -k regex:k_final_t -c 1 -o gpurun_out/prof_final30 python bench.py --config 1d_2e30 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 $P -k regex:k_rows -c 1 -o gpurun_out/prof_rows8192 python bench.py --config 2d_8192 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
for r in comb30 final30 rows8192; do
  ncu -i gpurun_out/prof_$r.ncu-rep --page source --csv > gpurun_out/prof_${r}_source.csv 2>&1
done
python tools/ncu_summary.py gpurun_out/prof_comb30.ncu-rep gpurun_out/prof_final30.ncu-rep gpurun_out/prof_rows8192.ncu-rep > gpurun_out/prof3.json
rm -f gpurun_out/prof_final30.ncu-rep gpurun_out/prof_rows8192.ncu-rep
