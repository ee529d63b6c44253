set -x
TILEFFT_COMB_F32=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
CASES='[["1d", 24], ["1d", 26], ["1d", 27]]' timeout 900 python tools/gpu/time_cfg.py '[{}, {"TILEFFT_COMB_F32": 1}, {"TILEFFT_DEBUG_COPYONLY": 1}, {"TILEFFT_COMB_F32": 1, "TILEFFT_DEBUG_COPYONLY": 1}]'
