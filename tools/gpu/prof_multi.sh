# ncu --set full on the passes of the 2^26 and 2^30 plans (one launch each).
timeout 900 ncu --set full --clock-control none --import-source on -c 3 -o gpurun_out/prof_2e26 \
  python bench.py --config 1d_2e26 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_2e26.ncu-rep > gpurun_out/prof_2e26.json
