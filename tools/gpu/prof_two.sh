timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_two -c 2 -o gpurun_out/prof_two \
  python bench.py --config 1d_2e26 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_two.ncu-rep > gpurun_out/prof_two.json
