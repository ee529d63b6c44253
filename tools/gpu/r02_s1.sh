#!/bin/bash
# headline kernel with one slot per warp, refilled after the exchange (more warps per SM) vs two slots
for v in 1 2 3; do
  TILEFFT_ROWS_S1=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "batched_1024 or fp32_within or device_path" 2>&1 | tail -1
done
for rep in 1 2; do
for v in 0 1 2 3; do
  TILEFFT_ROWS_S1=$v python bench.py --configs none --steps 200 --e2e-steps 0 --no-cpu-baseline --no-cufft | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('s1 $v', d['ms_per_step'], d['roofline']['pass_ms'])"
done
done
