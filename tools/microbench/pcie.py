"""PCIe H2D / D2H / bidirectional bandwidth from pinned memory (the e2e ceiling)."""
import torch, time
n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(f, reps=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
th = t(lambda: d.copy_(h, non_blocking=True)); td = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
tb = t(both)
print(f"H2D {n/th/1e9:.1f} GB/s  D2H {n/td/1e9:.1f} GB/s  bidir {2*n/tb/1e9:.1f} GB/s total ({tb*1e3:.2f} ms for 512 MiB each way)")
