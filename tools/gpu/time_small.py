"""Device time of back-to-back small transforms with the host launch cost hidden:
a spin kernel holds the stream while the K launches are queued (torch.cuda._sleep)."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1707_07263_b200 import _capi

def measure(fn, reps=200, hide=True):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if hide: torch.cuda._sleep(20_000_000)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

for v in json.loads(sys.argv[1]):
    for k in [k for k in os.environ if k.startswith("TILEFFT_")]: os.environ.pop(k)
    os.environ.update({k: str(x) for k, x in v.items()})
    for lg in json.loads(os.environ.get("LOGS", "[14, 16, 18, 19, 20, 21, 22]")):
        n = 1 << lg
        x = torch.randn(n, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
        dp = _capi.DevicePlan.create(n, 1, None, 8, _capi.MODE_FAST, None, 0)
        s = torch.cuda.current_stream().cuda_stream
        f = lambda: dp.exec_device(x.data_ptr(), y.data_ptr(), _capi.FORWARD, s)
        print(f"{v} 2^{lg} {dp.info()['factors']} launches {dp.info()['launches_per_exec']}: "
              f"queued {measure(f):.2f} us, host-driven {measure(f, hide=False):.2f} us", flush=True)
        dp.close()
