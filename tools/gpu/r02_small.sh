#!/bin/bash
# 2^20 (L2 flushed per step) and 2^18 x 4: small-transform paths (4-comb tiles, k_final_t) vs 16-comb TMA tiles + k_final_p (TILEFFT_SMALL_OFF=1)
mkdir -p gpurun_out
for rep in 1 2; do
for v in 0 1; do
  TILEFFT_SMALL_OFF=$v timeout 300 python bench.py --configs 1d_2e20 --steps 200 --warmup 5 --no-cpu-baseline --no-cufft --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['configs']['1d_2e20']; print('SMALL_OFF=$v 1d_2e20', r['ms_per_step'], r['roofline'].get('pass_ms'), d['clocks']['sm_mhz'])"
done; done
CASE_TIMEOUT=60 REPS=200 python tools/gpu/two_probe.py '[["1d", 20], ["1d", 21], ["1d", 19]]' '[{"TILEFFT_SMALL_OFF": 0}, {"TILEFFT_SMALL_OFF": 1}, {"TILEFFT_SMALL_OFF": 0}, {"TILEFFT_SMALL_OFF": 1}]'
