#!/bin/bash
# Final pass tile order: adjacent leading-digit chunks on consecutive tiles (TILEFFT_FINAL_CFIRST=1), parity + A/B

mkdir -p gpurun_out
TILEFFT_FINAL_CFIRST=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py -k "transposed_handover or multipass_inplace or 2e26_bench or 2e30_bench or fp32_within or inverse" -x -q > gpurun_out/fcfirst_tests.log 2>&1; tail -3 gpurun_out/fcfirst_tests.log
for rep in 1 2; do
for v in 0 1; do
  TILEFFT_FINAL_CFIRST=$v timeout 300 python bench.py --configs 1d_2e30,1d_2e26,1d_2e20 --steps 20 --warmup 3 --no-cpu-baseline --no-cufft --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for c in ('1d_2e30','1d_2e26','1d_2e20'):
    r=d['configs'][c]; print('CFIRST=$v', c, r['ms_per_step'], r['roofline'].get('pass_ms'), d['clocks']['sm_mhz'])"
done; done
