python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
python bench.py --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_batched_tma.csv python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rows -s 3 -c 1 -o gpurun_out/prof_batched_tma python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
