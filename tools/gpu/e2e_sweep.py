import time, torch, numpy as np, sys, os
sys.path.insert(0, '.')
from paper_1707_07263_b200 import _capi
import bench
n, b = 1024, 65536
x = torch.from_numpy(bench.splitmix_signal(n*b).view(np.float32)).pin_memory()
y = torch.empty_like(x).pin_memory()
for mb in [int(a) for a in sys.argv[1:]]:
    os.environ["TILEFFT_HOST_CHUNK_MB"] = str(mb)
    p = _capi.DevicePlan.create(n, b, None, 8, 0, None, 0)
    p.exec_host(x.data_ptr(), y.data_ptr())
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); p.exec_host(x.data_ptr(), y.data_ptr()); ts.append(time.perf_counter() - t0)
    print(mb, "MB chunks:", round(min(ts)*1e3, 3), "ms", round(np.median(ts)*1e3, 3))
    p.close()
