set -x
TILEFFT_ROWS_BULKSTORE=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "batched or fast_mode or device_path" 2>&1 | tail -1
for v in 0 1 0 1; do
  TILEFFT_ROWS_BULKSTORE=$v timeout 300 python bench.py --steps 200 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bulkstore $v', d['ms_per_step'], d['roofline']['frac'])"
done
