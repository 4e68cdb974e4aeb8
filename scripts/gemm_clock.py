"""Effective SM clock during back-to-back K2 launches (QARVD_GEMM_TRACE on the last one)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
M = 4680
name, n, k, no = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
spec = synth.LayerSpec(7, "l", n, k, M, no / k, 8.0)
w = synth.synth_weight(spec, seed=1)
plan = engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers)
L = engine.prepare_weights("l", w, plan)
x = synth.synth_activation(M, k, seed=3)
xq, sx, _ = engine.kernel_a_quantize_activation(x, L)
y = torch.empty((M, n), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n, L.k_pad,
                      L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                      None, 0, qb.BF16, y.data_ptr(), n, None, None, st)
for _ in range(int(sys.argv[5]) if len(sys.argv) > 5 else 200):  # sustained load first
    f()
os.environ["QARVD_GEMM_TRACE"] = "1"
f(); torch.cuda.synchronize()
