#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_plans.py -q -x -k "fast or 2e26 or 2e30 or inverse" 2>&1 | tail -1
export CASE_TIMEOUT=120 REPS=50
python tools/gpu/two_probe.py '[["1d", 30], ["1d", 26], ["1d", 24], ["1d", 22], ["1d", 20]]' '[{}]'
