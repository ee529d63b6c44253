#!/bin/bash
export CASE_TIMEOUT=60 REPS=300
for i in 1 2 3 4 5 6 7 8; do
python tools/gpu/two_probe.py '[["1d", 26]]' '[{"TILEFFT_TWO_1D": 1, "TILEFFT_TWO_D": 40, "TILEFFT_TWO_NSLOT": 56}]'
done
python tools/gpu/two_probe.py '[["2d", 8192, 8192], ["1d", 26]]' '[{}, {"TILEFFT_TWO_1D": 1}]'
for rep in 1 2; do
for t in 0 1 2; do
  TILEFFT_ROWS_DYN=$t python bench.py --configs none --steps 200 --e2e-steps 0 --no-cpu-baseline --no-cufft | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dyn $t', d['ms_per_step'], d['roofline']['pass_ms'])"
done
done
TILEFFT_ROWS_DYN=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "batched_1024 or fp32_within or inverse or device_path or two_streams" 2>&1 | tail -1
