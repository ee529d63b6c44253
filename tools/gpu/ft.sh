set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_twolevel.py tests/test_cpp_dropin.py -q -x 2>&1 | tail -2
CASES='[["1d", 22], ["1d", 24], ["1d", 26], ["1d", 30]]' timeout 900 python tools/gpu/time_cfg.py '[{}, {"TILEFFT_NO_FINAL_TMA": 1}]'
