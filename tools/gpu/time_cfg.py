"""Time device-resident transforms (1D and 2D) under env variants."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1707_07263_b200 as tf
from paper_1707_07263_b200 import _capi

def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

def run(v, cases):
    for k in list(os.environ):
        if k.startswith("TILEFFT_"): os.environ.pop(k)
    os.environ.update({k: str(x) for k, x in v.items()})
    for c in cases:
        if c[0] == "1d":
            n = 1 << c[1]
            x = torch.randn(n, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
            dp = _capi.DevicePlan.create(n, 1, None, 8, _capi.MODE_FAST, None, 0)
            us = timeit(lambda: dp.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, torch.cuda.current_stream().cuda_stream))
            print(f"{v} 1d 2^{c[1]} factors {dp.info()['factors']}: {us:.1f} us")
            dp.close()
        else:
            ny, nx = c[1], c[2]
            x = torch.randn(ny * nx, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
            dp = _capi.DevicePlan.create_2d(ny, nx, 1, 8, 0)
            us = timeit(lambda: dp.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, torch.cuda.current_stream().cuda_stream))
            print(f"{v} 2d {ny}x{nx} factors {dp.info()['factors']}: {us:.1f} us")
            dp.close()
        del x, y
        torch.cuda.empty_cache()

cases = [tuple(c) for c in json.loads(os.environ.get("CASES", "[[\"1d\", 24], [\"1d\", 26], [\"2d\", 8192, 8192]]"))]
for v in json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]:
    run(v, cases)
