"""PCIe ceiling for the e2e leg: pinned H2D alone, D2H alone, both at once (512 MiB each)."""
import time, torch
n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts)
def h2d():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
def chunked(ch=16 << 20):
    for o in range(0, n, ch):
        with torch.cuda.stream(s1): d_a[o:o + ch].copy_(h_in[o:o + ch], non_blocking=True)
        with torch.cuda.stream(s2): h_out[o:o + ch].copy_(d_b[o:o + ch], non_blocking=True)
for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both), ("both chunked 16MiB", chunked)]:
    s = t(fn)
    print(f"{name:20s} {s*1e3:8.2f} ms  {n/s/1e9:6.1f} GB/s per direction", flush=True)
