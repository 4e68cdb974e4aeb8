"""ffn.0 K2 (GELU epilogue) timing under epilogue diagnostics (QARVD_GEMM_DEBUG): 0 = normal,
128 = GELU without MUFU ops, 32 = math without stores, 16 = no tail."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, "%s")
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
M, n, k = 4680, 8960, 1536
spec = synth.LayerSpec(8, "l", n, k, M, 0.021, 8.0)
w = synth.synth_weight(spec, seed=1)
plan = engine.build_plan("l", k, qb.analyze_layer("l", w).aligned_outliers)
L = engine.prepare_weights("l", w, plan)
x = synth.synth_activation(M, k, seed=3)
xq, sx, _ = engine.kernel_a_quantize_activation(x, L)
y = torch.empty((M, n), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.call("qarvd_dual_gemm", xq.data_ptr(), L.k_pad, L.wq.data_ptr(), L.k_pad, M, n, L.k_pad,
                      L.k_outlier, sx.data_ptr(), L.scale_outlier32.data_ptr(), L.scale_normal32.data_ptr(),
                      None, qb.EPI_GELU, qb.BF16, y.data_ptr(), n, None, None, st)
for _ in range(5): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): f()
e1.record(); e1.synchronize()
print(round(e0.elapsed_time(e1) / 50 * 1e3, 1), "us")
''' % ROOT
for dbg in ["0", "128", "32", "16"]:
    env = dict(os.environ, QARVD_GEMM_DEBUG=dbg)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print("debug", dbg, r.stdout.strip() or r.stderr[-400:], flush=True)
