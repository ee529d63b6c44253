set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twolevel.py -q -x 2>&1 | tail -2
LOGS='[14, 16, 18, 20, 22, 24, 26]' timeout 600 python tools/gpu/time_small.py '[{"TILEFFT_NO_PDL": 1}, {}]'
CASES='[["2d", 8192, 8192], ["1d", 30]]' timeout 900 python tools/gpu/time_cfg.py '[{"TILEFFT_NO_PDL": 1}, {}]'
