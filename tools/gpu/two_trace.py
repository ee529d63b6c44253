"""Per-item timeline of one two-level column pass (TILEFFT_TWO_TRACE=1): where do items wait?"""
import ctypes, os, sys, json
import numpy as np
os.environ["TILEFFT_TWO_TRACE"] = "1"
import torch
sys.path.insert(0, os.getcwd())
from paper_1707_07263_b200 import _capi
ny = nx = 8192
dp = _capi.DevicePlan.create_2d(ny, nx, 1, 8, 0)
x = torch.randn(ny * nx, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
st = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    dp.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, st)
torch.cuda.synchronize()
lib = _capi.load() if hasattr(_capi, "load") else None
lib = ctypes.CDLL(os.path.join(os.getcwd(), "paper_1707_07263_b200", "libtilefft_b200.so"))
lib.tilefft_debug_two_trace.restype = ctypes.c_longlong
n = lib.tilefft_debug_two_trace(None, 0)
buf = np.zeros(n // 8, dtype=np.uint64)
lib.tilefft_debug_two_trace(buf.ctypes.data_as(ctypes.c_void_p), n)
T = buf.reshape(-1, 8).astype(np.int64)
t0 = T[:, 0].min()
T[:, :6] -= t0
isA = T[:, 7] == 1
span = T[:, 5].max()
print(f"items {len(T)}  span {span/1e3:.1f} us  (diag={os.environ.get('TILEFFT_TWO_DIAG', '0')})")
names = ["claim->dep", "dep->empty", "empty->full(TMA)", "full->slot free", "slot free->done"]
for kind, m in (("A", isA), ("B", ~isA)):
    d = np.diff(T[m][:, :6], axis=1) / 1e3
    print(kind, " ".join(f"{nm}: med {np.median(d[:, i]):.2f} p90 {np.percentile(d[:, i], 90):.2f}" for i, nm in enumerate(names)))
# per-SM: time the compute warps spend idle between items (done of k -> full of k+1 on the same CTA)
idle = []
busy = []
for c in range(int(T[:, 6].max()) + 1):
    r = T[T[:, 6] == c]
    r = r[np.argsort(r[:, 3])]
    busy.append(((r[:, 5] - r[:, 3]).sum()) / 1e3)
    idle.append(span / 1e3 - busy[-1])
print(f"per-CTA compute busy (full->done summed) median {np.median(busy):.1f} us, idle median {np.median(idle):.1f} us")
# rate over time
h, _ = np.histogram(T[:, 5], bins=20)
print("items done per 5% of span:", h.tolist())
