"""Stream-K vs data-parallel K2 on the FFN-down shape: event timings (L2 flushed) and a CTA-0 trace."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
M, n, k = 4680, 1536, 8960
spec = synth.LayerSpec(7, "l", n, k, M, 0.021, 8.0)
w = synth.synth_weight(spec, seed=1)
plan = engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers)
L = engine.prepare_weights("l", w, plan)
x = synth.synth_activation(M, k, seed=3)
xq, sx, _ = engine.kernel_a_quantize_activation(x, L)
y = torch.empty((M, n), dtype=torch.bfloat16, device="cuda")
nb = int(_lib.load().qarvd_dual_gemm_workspace_size(M, n, L.k_pad, L.k_outlier))
ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device="cuda")
print("workspace bytes", nb, "k_pad", L.k_pad, "k_o", L.k_outlier)
st = torch.cuda.current_stream().cuda_stream
dp = lambda: _lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n, L.k_pad,
                       L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                       None, 0, qb.BF16, y.data_ptr(), n, None, None, st)
sk = lambda: _lib.call("qarvd_dual_gemm_ws", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n, L.k_pad,
                       L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                       None, 0, y.data_ptr(), n, ws.data_ptr(), ws.numel(), st)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, f in (("dp", dp), ("sk", sk), ("dp", dp), ("sk", sk)):
    for _ in range(3): f()
    ts = []
    for _ in range(20):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, "median us", round(float(np.median(ts)), 1), "min", round(min(ts), 1))
os.environ["QARVD_GEMM_TRACE"] = "1"
for cta in os.environ.get("CTAS", "0").split(","):
    os.environ["QARVD_GEMM_TRACE_CTA"] = cta
    for name, f in (("dp", dp), ("sk", sk)):
        print("=== trace", name, "cta", cta); sys.stdout.flush()
        f(); torch.cuda.synchronize(); sys.stdout.flush()
