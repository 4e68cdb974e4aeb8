"""Per-CTA start / end times (globaltimer) of one K2 launch (QARVD_GEMM_DEBUG=128): how the
kernel's duration splits into CTA launch skew, per-CTA work and the tail."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
M = 4680
n, k, no, epi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
spec = synth.LayerSpec(7, "l", n, k, M, no / k, 8.0)
w = synth.synth_weight(spec, seed=1)
L = engine.prepare_weights("l", w, engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers))
xq, sx, _ = engine.kernel_a_quantize_activation(synth.synth_activation(M, k, seed=3), L)
y = torch.empty((M, n), dtype=torch.bfloat16, device="cuda")
f = lambda: _lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n, L.k_pad,
                      L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                      None, epi, qb.BF16, y.data_ptr(), n, None, None, None)
for _ in range(5):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); f(); e1.record(); torch.cuda.synchronize()
print(f"N={n} K={k}: event-timed {e0.elapsed_time(e1)*1e3:.1f} us")
os.environ["QARVD_GEMM_DEBUG"] = "128"
lib = _lib.load()
for rep in range(2):
    f(); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 296)()
    assert lib.qarvd_debug_cta_times(buf, 148) == 0
    t = np.array(buf[:], dtype=np.int64).reshape(148, 2)
    t0 = t[:, 0].min()
    s, e = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    print(f"  start: min 0 median {np.median(s):.2f} max {s.max():.2f} us | end: min {e.min():.2f} "
          f"median {np.median(e):.2f} max {e.max():.2f} us | busy per CTA median {np.median(e - s):.2f} us")
    order = np.argsort(s)
    print("  latest starters:", [(int(i), round(float(s[i]), 2)) for i in order[-6:]])
    print("  latest finishers:", [(int(i), round(float(e[i]), 2)) for i in np.argsort(e)[-6:]])
del os.environ["QARVD_GEMM_DEBUG"]
