set -x
TILEFFT_SMALL_F=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fast_mode" 2>&1 | tail -1
TILEFFT_SMALL_F=8 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fast_mode" 2>&1 | tail -1
LOGS='[14, 16, 18, 19, 20]' timeout 600 python tools/gpu/time_small.py '[{}, {"TILEFFT_SMALL_F": 2}, {"TILEFFT_SMALL_F": 8}]'
