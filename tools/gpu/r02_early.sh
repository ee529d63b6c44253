#!/bin/bash
# EARLY slot refill A/B for the headline kernel + the distributed graph-capture test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_distributed.py -m gpu -x -q 2>&1 | grep -E "Error|error:|passed|failed" | head -20
for t in 1 2 3; do
  TILEFFT_ROWS_EARLY=$t timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "batched_1024 or fp32_within or inverse or device_path" 2>&1 | tail -1
done
for rep in 1 2; do
for t in 0 1 2 3; do
  TILEFFT_ROWS_EARLY=$t python bench.py --configs none --steps 200 --e2e-steps 0 --no-cpu-baseline --no-cufft | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('early $t', d['ms_per_step'], d['roofline']['pass_ms'])"
done
done
