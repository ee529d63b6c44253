# two-level pass: parity + timing + launch list
timeout 900 python -m pytest tests/test_gpu_twolevel.py -x -q 2>&1 | tail -15
for c in 1d_2e26 2d_8192; do timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:40], d['ms_per_step'], d['value'], d['roofline']['frac'], d['config'].get('device_factors'))"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 1d_2e26 2d_8192; do
  timeout 600 ncu --metrics $M --clock-control none -c 6 --csv --log-file gpurun_out/launches_two_$c.csv \
    python bench.py --config $c --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/launches_two_$c.csv
done
