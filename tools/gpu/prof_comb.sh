ncu --set full --clock-control none --import-source on -k regex:k_comb -s 3 -c 1 -o gpurun_out/prof_comb512 python bench.py --config 1d_2e26 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_final -s 1 -c 1 -o gpurun_out/prof_final256 python bench.py --config 1d_2e26 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_comb -s 3 -c 1 -o gpurun_out/prof_comb_2d python bench.py --config 2d_8192 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_2d.csv python bench.py --config 2d_8192 --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
