"""cuBLAS DGEMM throughput on this B200 (the denominator for K7's f64 GEMM share)."""
import json
import torch

out = {}
for (m, n, k) in ((8192, 8192, 8192), (12480, 1536, 1536), (1536, 1536, 12480), (1560, 1536, 1536),
                  (1536, 1536, 1560)):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[f"{m}x{n}x{k}"] = {"ms": ms, "tflops": 2.0 * m * n * k / ms / 1e9}
print(json.dumps(out))
