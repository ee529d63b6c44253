set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
CASES='[["1d", 24], ["1d", 26], ["1d", 30]]' timeout 900 python tools/gpu/time_cfg.py '[{"TILEFFT_COMB_L2PF": 0}, {}, {"TILEFFT_COMB_L2PF": 0, "TILEFFT_DEBUG_COPYONLY": 1}, {"TILEFFT_DEBUG_COPYONLY": 1}]'
