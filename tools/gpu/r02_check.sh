#!/bin/bash
# full GPU suite, smoke, default bench line (all configs), two-level timing with the dependency-wait watchdog
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -2 gpurun_out/bench_default.err
python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
def show(n, r):
    rf = r.get('roofline') or {}
    print(n, r.get('ms_per_step'), r.get('value'), 'kfrac', rf.get('frac'), 'step', (rf.get('step') or {}).get('frac'), rf.get('pass_ms'), 'cufft', (r.get('cufft') or {}).get('ms_per_step'), r.get('error'))
show('batched1024', d)
for k, v in d.get('configs', {}).items(): show(k, v)
print(d['clocks'])
PY
CASE_TIMEOUT=60 REPS=300 python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_1D": 1}, {"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 40, "TILEFFT_TWO_NSLOT": 56}]'
