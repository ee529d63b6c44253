#!/bin/bash
TILEFFT_FINAL_WS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast_mode or inverse" 2>&1 | tail -1
for i in 1 2 3; do
python - <<'PY'
import os, sys, torch, subprocess
PY
for ws in 0 1; do
TILEFFT_FINAL_WS=$ws python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1707_07263_b200 import _capi
for lg in (26, 28, 30):
    n = 1 << lg
    dp = _capi.DevicePlan.create(n, 1, None, 8, _capi.MODE_FAST, None, 0)
    x = torch.randn(n, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
    dp.exec_timed(x.data_ptr(), y.data_ptr(), reps=2)
    ms = dp.exec_timed(x.data_ptr(), y.data_ptr(), reps=10)
    print("ws", os.environ["TILEFFT_FINAL_WS"], lg, [round(m, 4) for m in ms], flush=True)
    del x, y; dp.close(); torch.cuda.empty_cache()
PY
done
done
