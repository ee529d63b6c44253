#!/bin/bash
# 32-row final tiles (256-byte output lines) for L <= 512 (TILEFFT_FINAL_F32=1) vs 16-row tiles, chunk-first order: parity, A/B
mkdir -p gpurun_out
TILEFFT_FINAL_F32=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py -k "transposed_handover or multipass_inplace or 2e26_bench or fp32_within or inverse" -x -q > gpurun_out/f32_tests.log 2>&1; tail -3 gpurun_out/f32_tests.log
for rep in 1 2; do
CASE_TIMEOUT=120 REPS=30 python tools/gpu/two_probe.py '[["1d", 26], ["1d", 25], ["1d", 24]]' '[{"TILEFFT_FINAL_F32": 0}, {"TILEFFT_FINAL_F32": 1}]'
CASE_TIMEOUT=120 REPS=10 python tools/gpu/two_probe.py '[["1d", 28], ["1d", 29]]' '[{"TILEFFT_FINAL_F32": 0}, {"TILEFFT_FINAL_F32": 1}]'
done
for v in 0 1; do
  TILEFFT_FINAL_F32=$v timeout 300 python bench.py --configs 1d_2e26 --steps 50 --warmup 3 --no-cpu-baseline --no-cufft --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['configs']['1d_2e26']; print('F32=$v 1d_2e26', r['ms_per_step'], r['roofline'].get('pass_ms'), d['clocks']['sm_mhz'])"
done
