#!/bin/bash
# register-resident stage roots for the headline kernel (A/B) + the device-barrier distributed tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_distributed.py -m gpu -x -q 2>&1 | tail -5
for t in 1 2; do
  TILEFFT_ROWS_TWR=$t timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "batched_1024 or fp32_within or inverse or device_path" 2>&1 | tail -1
done
for rep in 1 2; do
for t in 0 1 2; do
  TILEFFT_ROWS_TWR=$t python bench.py --configs none --steps 200 --e2e-steps 0 --no-cpu-baseline --no-cufft | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('twr $t', d['ms_per_step'], d['roofline']['pass_ms'])"
done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
TILEFFT_ROWS_TWR=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_rows_tma -s 3 -c 1 -o /tmp/prof_twr python bench.py --configs none --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-cufft > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof_twr.ncu-rep > gpurun_out/ncu_rows_tma_twr.json
ncu -i /tmp/prof_twr.ncu-rep --page source --csv > /tmp/src_twr.csv 2>&1
python tools/ncu_source_top.py /tmp/src_twr.csv 40 > gpurun_out/ncu_rows_tma_twr_top_sass.txt
