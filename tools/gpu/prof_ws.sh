# ncu --set full of the warp-specialised two-level pass in the 2D 8192^2 config
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_two_ws -c 1 -o gpurun_out/prof_ws \
  python bench.py --config 2d_8192 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_ws.ncu-rep > gpurun_out/prof_ws.json
ncu -i gpurun_out/prof_ws.ncu-rep --page source --csv > gpurun_out/prof_ws_source.csv 2>&1
ncu -i gpurun_out/prof_ws.ncu-rep --page details --csv > gpurun_out/prof_ws_details.csv 2>&1
