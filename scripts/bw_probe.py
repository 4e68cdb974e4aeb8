"""Achievable HBM traffic for K1's shape: torch elementwise kernels on the same bytes
(84 MB bf16 read + 42 MB int8 write), L2 flushed between reps; device times via events."""
import torch

M, K = 4680, 8960
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out8 = torch.empty(M, K, dtype=torch.int8, device="cuda")
out16 = torch.empty_like(x)


def t(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for name, fn, nbytes in [
    ("bf16->int8 cast (84R+42W MB)", lambda: out8.copy_(x), M * K * 3),
    ("bf16 copy (84R+84W MB)", lambda: out16.copy_(x), M * K * 4),
    ("bf16 sum (84R MB)", lambda: x.sum(), M * K * 2),
]:
    us = t(fn)
    print(f"{name:32s} {us:7.1f} us  {nbytes / us / 1e3:7.0f} GB/s")
