"""K1 marginal cost: time of 1 vs 2 back-to-back launches after an L2 flush (the second
launch pays no shared-memory carveout switch), and after a large-smem GEMM."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3
out = {}
M = 4680
for k in (1536, 8960):
    plan = engine.build_plan("l", k, list(range(0, k, k // 32))[:32])
    g = torch.from_numpy(plan.gather).cuda()
    x = synth.synth_activation(M, k, seed=3)
    xq = torch.empty((M, plan.k_pad), dtype=torch.int8, device="cuda")
    sx = torch.empty(M, dtype=torch.float32, device="cuda")
    f = lambda: _lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, M, k, k, g.data_ptr(), plan.k_pad, 0, 0.0, 8,
                          xq.data_ptr(), plan.k_pad, sx.data_ptr(), None, None, st)
    t1 = timeit(f)
    t2 = timeit(lambda: (f(), f()))
    t3 = timeit(lambda: (f(), f(), f()))
    out[f"k{k}"] = {"one_us": t1, "two_us": t2, "three_us": t3, "marginal_us": (t3 - t1) / 2,
                    "bytes": M * (k * 2 + plan.k_pad + 4)}
    out[f"k{k}"]["marginal_gbs"] = out[f"k{k}"]["bytes"] / (out[f"k{k}"]["marginal_us"] * 1e-6) / 1e9
print(json.dumps(out, indent=1))
