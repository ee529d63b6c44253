#!/bin/bash
timeout 1500 python -m pytest tests/test_distributed.py tests/test_gpu_bench_plans.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_ip.json 2> gpurun_out/bench_ip.err; python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_ip.json').read().strip().splitlines()[-1])
def show(n, r):
    rf = r.get('roofline') or {}
    print(n, r.get('ms_per_step'), r.get('value'), 'kfrac', rf.get('frac'), 'step', (rf.get('step') or {}).get('frac'), rf.get('pass_ms'), 'cufft', (r.get('cufft') or {}).get('ms_per_step'))
show('batched1024', d)
for k, v in d.get('configs', {}).items(): show(k, v)
print(d['clocks'])
PY
