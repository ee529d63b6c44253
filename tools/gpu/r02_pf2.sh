#!/bin/bash
# Long-row pass with an extra half-row landing zone (k_rows_pf2, TILEFFT_ROWS_PF2=1) vs k_rows_pf: parity, A/B
mkdir -p gpurun_out
TILEFFT_ROWS_PF2=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py tests/test_gpu_twolevel.py -k "long_rows or 2d or 8192" -x -q > gpurun_out/pf2_tests.log 2>&1; tail -3 gpurun_out/pf2_tests.log
for rep in 1 2; do
for v in 0 1; do
  TILEFFT_ROWS_PF2=$v timeout 300 python bench.py --configs 2d_8192 --steps 50 --warmup 3 --no-cpu-baseline --no-cufft --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for c in ('2d_8192',):
    r=d['configs'][c]; print('PF2=$v', c, r['ms_per_step'], r['roofline'].get('pass_ms'), d['clocks']['sm_mhz'])"
done; done
CASE_TIMEOUT=120 REPS=50 python tools/gpu/two_probe.py '[["2d", 4096, 4096], ["2d", 2048, 2048], ["2d", 16384, 8192]]' '[{"TILEFFT_ROWS_PF2": 0}, {"TILEFFT_ROWS_PF2": 1}, {"TILEFFT_ROWS_PF2": 0}, {"TILEFFT_ROWS_PF2": 1}]'
