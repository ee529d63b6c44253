set -x
python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -4
python bench.py > gpurun_out/bench_batched.json 2> gpurun_out/bench_err.txt; cat gpurun_out/bench_batched.json; tail -3 gpurun_out/bench_err.txt
for c in 1d_2e20 1d_2e26 2d_8192 1d_2e30; do python bench.py --config $c --no-cpu-baseline --e2e-steps 2 --steps 50 2>&1 | tail -1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_batched.csv python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_2e26.csv python bench.py --config 1d_2e26 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rows -s 3 -c 1 -o gpurun_out/prof_batched python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
