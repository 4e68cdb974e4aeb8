"""Traced fused-quantizer K2 launches (QARVD_GEMM_TRACE): per-tile clocks of chosen CTAs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
M, n, k, no = 4680, 8960, 1536, 32
spec = synth.LayerSpec(7, "l", n, k, M, no / k, 8.0)
w = synth.synth_weight(spec, seed=1)
plan = engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers)
L = engine.prepare_weights("l", w, plan)
x = synth.synth_activation(M, k, seed=3)
xq, sx, _ = engine.kernel_a_quantize_activation(x, L)
q = torch.empty((M, n), dtype=torch.int8, device="cuda")
s = torch.empty(M, dtype=torch.float32, device="cuda")
ws = torch.zeros(int(_lib.load().qarvd_dual_gemm_quant_workspace_size(M)), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.call("qarvd_dual_gemm_quant", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n, L.k_pad,
                      L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                      None, qb.EPI_GELU, qb.ACT_PER_TOKEN, 0.0, 8, q.data_ptr(), n, s.data_ptr(), None, None,
                      ws.data_ptr(), ws.numel(), st)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); f(); e1.record(); torch.cuda.synchronize()
print("fused K2 %.1f us" % (e0.elapsed_time(e1) * 1e3))
for cta in sys.argv[1:] or ["0", "141"]:
    os.environ["QARVD_GEMM_TRACE"] = "1"
    os.environ["QARVD_GEMM_TRACE_CTA"] = cta
    print("=== CTA", cta); sys.stdout.flush()
    f(); torch.cuda.synchronize()
    del os.environ["QARVD_GEMM_TRACE"]
