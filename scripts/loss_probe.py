"""Eq. 5 kernel: accuracy vs the reference on small cases, and timing at Wan calibration shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import engine, calibrate, synth
import test_gpu_parity as T

for case in [(256, 512, 32, (40, 77, 13)), (300, 1536, 64, (200, 129)), (136, 320, 0, (128,)), (192, 896, 96, (1, 255, 256, 3))]:
    ref, layer, wd, batch, cw, _ = T._ref_loss_case(*case, seed=case[0] + case[1])
    loss = calibrate.weighted_loss(batch, layer, wd, cw, ref["act_scale"])
    print("case", case[:3], "rel err", abs(loss - ref["loss"]) / ref["loss"])

for (n, k) in [(1536, 1536), (8960, 1536), (1536, 8960)]:
    spec = [s for s in synth.wan_registry(blocks=1) if s.out_dim == n and s.in_dim == k][0]
    w = synth.synth_weight(spec, seed=1)
    rep = qb.analyze_layer(spec.name, w)
    plan = engine.build_plan(spec.name, k, rep.aligned_outliers)
    layer = engine.prepare_weights(spec.name, w, plan)
    xs = torch.cat([synth.synth_activation(1560, k, seed=3, frame=f) for f in range(21)])
    m = xs.shape[0]
    xq, s32, _ = engine.kernel_a_quantize_activation(xs, layer, qb.ACT_PER_TENSOR, static_scale=float(xs.float().abs().max()) / 127)
    rows = np.arange(22, dtype=np.int64) * 1560
    chunks = np.arange(1, 22, dtype=np.int64)
    cw = calibrate.weighting_strategy("heuristic_exp", 21)
    wsb = int(qb._lib.load().qarvd_weighted_loss_workspace(m, n, 21))
    ws = torch.empty(wsb // 8, dtype=torch.float64, device="cuda")
    err = torch.empty(21, dtype=torch.float64, device="cuda")
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    def run():
        qb._lib.call("qarvd_weighted_loss", xs.data_ptr(), k, w.data_ptr(), k, xq.data_ptr(), layer.k_pad,
                     layer.wq.data_ptr(), layer.k_pad, m, n, k, layer.k_pad, layer.k_outlier, s32.data_ptr(),
                     layer.scale_outlier32.data_ptr(), layer.scale_normal32.data_ptr(), rows.ctypes.data,
                     chunks.ctypes.data, 21, cw.ctypes.data, 21, err.data_ptr(), loss.data_ptr(), ws.data_ptr(), wsb, 0)
    for _ in range(3): run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    fl = 2.0 * m * n * k
    print(f"loss {n}x{k} M={m}: {ms:.3f} ms  bf16 {fl/ms/1e9:.0f} TF/s + int8 {2*m*n*layer.k_pad/ms/1e9:.0f} TOPS"
          f"  (ideal at 1635 TF bf16 + 3270 TOPS int8: {(fl/1635e12 + 2*m*n*layer.k_pad/3270e12)*1e3:.3f} ms)")
    # cuBLAS bf16 reference point: the target GEMM alone
    t = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    for _ in range(3): torch.matmul(xs, w.t(), out=t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): torch.matmul(xs, w.t(), out=t)
    e1.record(); e1.synchronize()
    print(f"   cuBLAS bf16 X W^T alone: {e0.elapsed_time(e1)/10:.3f} ms")
