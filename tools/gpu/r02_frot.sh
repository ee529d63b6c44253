#!/bin/bash
# Final pass: rotate each CTA's store order over k (TILEFFT_FINAL_ROT multiplier, 0 = off; variant removed) -- A/B
mkdir -p gpurun_out
for rep in 1 2; do
for v in 0 1 7; do
  TILEFFT_FINAL_ROT=$v timeout 300 python bench.py --configs 1d_2e30,1d_2e26 --steps 20 --warmup 3 --no-cpu-baseline --no-cufft --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for c in ('1d_2e30','1d_2e26'):
    r=d['configs'][c]; print('ROT=$v', c, r['ms_per_step'], r['roofline'].get('pass_ms'), d['clocks']['sm_mhz'])"
done; done
