"""PCIe floor for the e2e path: 14.4 MB pinned H2D, D2H, and both concurrently."""
import torch
n = 4680 * 1536
xh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
yh = torch.empty(n, dtype=torch.bfloat16).pin_memory()
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
yd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
import time
def t(fn, reps=50):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    ts.sort(); return ts[len(ts) // 2] * 1e6
def h2d():
    with torch.cuda.stream(s1): xd.copy_(xh, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): yh.copy_(yd, non_blocking=True)
def both():
    h2d(); d2h()
for name, fn in [("H2D 14.4MB", h2d), ("D2H 14.4MB", d2h), ("both concurrently", both)]:
    us = t(fn); print(f"{name:20s} {us:7.1f} us  {n*2/us/1e3:6.1f} GB/s per direction")
