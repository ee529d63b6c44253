set -x
timeout 600 python -m pytest tests/test_gpu_twolevel.py -q -x 2>&1 | tail -2
CASES='[["2d", 8192, 8192], ["2d", 4096, 4096]]' timeout 900 python tools/gpu/time_cfg.py '[{}, {"TILEFFT_TWO_WS": 0}, {"TILEFFT_TWO_1D": 1}]'
CASES='[["1d", 24], ["1d", 26]]' timeout 900 python tools/gpu/time_cfg.py '[{"TILEFFT_TWO_1D": 1}]'
