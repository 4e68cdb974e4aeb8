"""K1 device time vs L2 state: no flush / 256 MiB write flush / write + clean-read flush (bench
mode), next to a plain torch copy of the same bytes under the same flush."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import engine, synth

torch.cuda.set_device(0)
M = 4680
wbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rbuf = torch.ones(64 << 20, dtype=torch.int32, device="cuda")
sink = torch.empty((), dtype=torch.int64, device="cuda")


def flush(mode):
    if mode >= 1:
        wbuf.fill_(1)
    if mode >= 2:
        sink.copy_(rbuf.sum())


def timeit(fn, mode, reps=30):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush(mode)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


for name, k, n in (("x (1536, gathered)", 1536, 1536), ("x (1536, plan order)", 1536, 1537),
                    ("U (8960, plan order)", 8960, 1536)):
    spec = synth.LayerSpec(7, "l", n, k, M, 0.021, 8.0)
    w = synth.synth_weight(spec, seed=1)
    L = engine.prepare_weights("l", w, engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers))
    x = synth.synth_activation(M, k, seed=3)
    xq = torch.empty((M, L.k_pad), dtype=torch.int8, device="cuda")
    sx = torch.empty(M, dtype=torch.float32, device="cuda")
    g = L.gather_dev if n == 1536 and k == 1536 else None
    kout = L.k_pad if g is not None else k
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: qb._lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, M, k, k, None if g is None else g.data_ptr(),
                             kout, qb.ACT_PER_TOKEN, 0.0, 8, xq.data_ptr(), kout, sx.data_ptr(), None, None, st)
    y = torch.empty_like(x)
    c = lambda: y.copy_(x)
    for mode in (0, 1, 2):
        print(f"{name}: flush {mode}: K1 {timeit(f, mode):6.1f} us   torch copy {timeit(c, mode):6.1f} us")
