#!/bin/bash
# Transposed pass-0 -> pass-1 hand-over (CombArgs::t_l2): parity tests, then A/B timing (TILEFFT_TSTORE=0 vs default/forced)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "transposed_handover or multipass_inplace" tests/test_gpu_bench_plans.py -k "transposed_handover or multipass_inplace or 2e30_bench" -x -q > gpurun_out/tstore_tests.log 2>&1; tail -3 gpurun_out/tstore_tests.log
for v in 0 -1 0 -1; do
  TILEFFT_TSTORE=$v timeout 300 python bench.py --configs 1d_2e30 --steps 20 --warmup 3 --no-cpu-baseline --no-cufft --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['configs']['1d_2e30']; print('TSTORE=$v 2^30', r['ms_per_step'], r['roofline'].get('pass_ms'), d.get('clocks'))"
done
CASE_TIMEOUT=120 REPS=20 python tools/gpu/two_probe.py '[["1d", 28], ["1d", 29], ["1d", 27], ["1d", 26]]' '[{"TILEFFT_TSTORE": 0}, {"TILEFFT_TSTORE": 1}, {"TILEFFT_TSTORE": 0}, {"TILEFFT_TSTORE": 1}]'
