"""K1 team-shape sweep for the K=1536 gathered quantize (FFN x) and the K=8960 plan-order one."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, "%s")
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
M = 4680
res = {}
for k in (1536, 8960):
    plan = engine.build_plan("l", k, list(range(0, k, k // 32))[:32])
    g = torch.from_numpy(plan.gather).cuda() if k == 1536 else None
    kout = plan.k_pad if k == 1536 else k
    x = synth.synth_activation(M, k, seed=3)
    xq = torch.empty((M, kout), dtype=torch.int8, device="cuda")
    sx = torch.empty(M, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, M, k, k, None if g is None else g.data_ptr(), kout, 0, 0.0, 8, xq.data_ptr(), kout, sx.data_ptr(), None, None, st)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3): f()
    ts = []
    for _ in range(30):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    res[k] = float(np.median(ts))
print(res)
''' % ROOT
for shape in ["default", "1x1", "1x2", "2x2", "2x3", "4x2", "4x3", "6x3", "7x3", "8x3"]:
    env = dict(os.environ)
    if shape != "default":
        env["QARVD_K1_SHAPE"] = shape
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print(shape, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:], flush=True)
