#!/bin/bash
# Final pass with 16-byte shared loads / global stores (two outputs per lane; TILEFFT_FINAL_VEC=1): parity, A/B;
# then the layout probe with 256-byte lines (tools/microbench/comb_layout.cu)
mkdir -p gpurun_out
TILEFFT_FINAL_VEC=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py -k "transposed_handover or multipass_inplace or 2e26_bench or 2e30_bench or fp32_within or inverse" -x -q > gpurun_out/fvec_tests.log 2>&1; tail -3 gpurun_out/fvec_tests.log
for rep in 1 2; do
for v in 0 1; do
  TILEFFT_FINAL_VEC=$v timeout 300 python bench.py --configs 1d_2e30,1d_2e26,1d_2e20 --steps 20 --warmup 3 --no-cpu-baseline --no-cufft --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for c in ('1d_2e30','1d_2e26','1d_2e20'):
    r=d['configs'][c]; print('VEC=$v', c, r['ms_per_step'], r['roofline'].get('pass_ms'), d['clocks']['sm_mhz'])"
done; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gpurun_out/comb_layout tools/microbench/comb_layout.cu
timeout 300 gpurun_out/comb_layout 2>&1 | tee gpurun_out/comb_layout256.txt
