"""K1 timing probe: full kernel vs QARVD_K1_DEBUG=1 (no code loop), warm vs cold L2, grid sweep."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def timeit(fn, reps=20, do_flush=True):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        if do_flush: flush.fill_(1)
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
    for dbg in ("0", "1"):
        os.environ["QARVD_K1_DEBUG"] = dbg
        out[f"k{k}_dbg{dbg}_cold_us"] = timeit(f)
        out[f"k{k}_dbg{dbg}_warm_us"] = timeit(f, do_flush=False)
    os.environ["QARVD_K1_DEBUG"] = "0"
    # plain copy of the same bytes for reference
    y = torch.empty_like(x)
    out[f"k{k}_torch_copy_cold_us"] = timeit(lambda: y.copy_(x))
print(json.dumps(out, indent=1))
