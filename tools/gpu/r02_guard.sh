#!/bin/bash
timeout 600 python -m pytest tests/test_capi.py -q 2>&1 | tail -2
# 2^30 pass times vs 2^28 (TLB hypothesis for pass 0: rows 8 MB apart at 2^30, 2 MB at 2^28)
python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1707_07263_b200 import _capi
for lg in (26, 28, 30):
    n = 1 << lg
    dp = _capi.DevicePlan.create(n, 1, None, 8, _capi.MODE_FAST, None, 0)
    x = torch.randn(n, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
    ms = dp.exec_timed(x.data_ptr(), y.data_ptr(), reps=5)
    print(lg, dp.info()["factors"], [round(m, 4) for m in ms], "GB/s per pass", [round(16 * n / (m * 1e-3) / 1e9) for m in ms])
    del x, y; dp.close(); torch.cuda.empty_cache()
PY
