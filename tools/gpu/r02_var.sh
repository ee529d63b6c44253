#!/bin/bash
# north-star prototypes on the headline kernel: warp-shuffle exchange (1), 128-bit stores (2), both (3)
for v in 1 2 3; do
  TILEFFT_ROWS_VAR=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "batched_1024 or fp32_within or inverse or device_path" 2>&1 | tail -1
done
for rep in 1 2; do
for v in 0 1 2 3; do
  TILEFFT_ROWS_VAR=$v python bench.py --configs none --steps 200 --e2e-steps 0 --no-cpu-baseline --no-cufft | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('var $v', d['ms_per_step'], d['roofline']['pass_ms'])"
done
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
for v in 0 1 2 3; do
  TILEFFT_ROWS_VAR=$v timeout 300 ncu --metrics $M --clock-control none -k regex:k_rows_tma -s 3 -c 1 --csv --log-file gpurun_out/var_$v.csv python bench.py --configs none --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-cufft > /dev/null 2>&1
  grep -E "inst_executed|wavefronts|duration" gpurun_out/var_$v.csv | awk -F'","' -v v=$v '{print "var", v, $(NF-2), $NF}'
done
