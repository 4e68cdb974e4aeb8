"""Small-shape pass over every product kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):  compute-sanitizer --tool racecheck python scripts/sanitize_driver.py
K1 (register, slot-ring, bulk-staged), K2 (bf16 + GELU epilogue, f64, f64 slices, pmax),
K3 / K5 (analyze + prepare), K4 (percentile search), K6 (Eq. 5 loss), K7 (AdaRound, a few
iterations), the C-ABI linear handle and chain."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import calibrate, engine, synth
from paper_2605_21072_b200.pipeline import QuantizedChain

torch.cuda.set_device(0)
torch.manual_seed(0)
M, D, F = 192, 256, 640

spec0 = synth.LayerSpec(0, "ffn.0", F, D, M, 0.05, 8.0)
spec2 = synth.LayerSpec(0, "ffn.2", D, F, M, 0.05, 8.0)
w0 = synth.synth_weight(spec0, seed=1)
w2 = synth.synth_weight(spec2, seed=2)
# K3 (+ K5 through prepare_weights)
r0, r2 = qb.analyze_layer("ffn.0", w0), qb.analyze_layer("ffn.2", w2)
L0 = engine.prepare_weights("ffn.0", w0, engine.build_plan("ffn.0", D, r0.aligned_outliers))
L2 = engine.prepare_weights("ffn.2", w2, engine.build_plan("ffn.2", F, r2.aligned_outliers))
x = synth.synth_activation(M, D, seed=3)
# K1 (gathered) + K2 (bf16), one linear
y = engine.quantized_layer_forward(L0, x)
# K1 variants
for bulk in ("0", "1"):
    os.environ["QARVD_K1_BULK"] = bulk
    engine.kernel_a_quantize_activation(x, L0)
    u = synth.synth_activation(M, F, seed=4)
    xq = torch.empty((M, F), dtype=torch.int8, device="cuda")
    qb._lib.call("qarvd_quantize_act", u.data_ptr(), qb.BF16, M, F, F, None, F, qb.ACT_PER_TOKEN, 0.0, 8,
                 xq.data_ptr(), F, None, None, None, None)
os.environ["QARVD_K1_BULK"] = "0"
# the FFN chain (GELU epilogue, folded K1, pmax fusion) and the C-ABI host chain
for fuse in (False, True):
    ch = QuantizedChain([L0, L2], M, epilogues=[qb.EPI_GELU, qb.EPI_NONE], fuse_rowmax=fuse)
    ch.x.copy_(x)
    ch.launch()
hs = [engine.LinearHandle(ch.layers[0], qb.EPI_GELU), engine.LinearHandle(ch.layers[1])]
xh = x.cpu().pin_memory()
yh = torch.empty((M, D), dtype=torch.bfloat16).pin_memory()
for _ in range(3):  # eager, capture, replay
    engine.chain_forward_host(hs, xh, yh)
for h in hs:
    h.close()
# K2 f64 epilogue and the K7 slice products + K4 + K6 + K7 through calibrate_layer
frames, rows = 3, 64
xs = [synth.synth_activation(rows, D, seed=10 + f, frame=f).double() for f in range(frames)]
act = max(float(t.abs().max()) for t in xs) / 127.0
cw = calibrate.weighting_strategy("heuristic_exp", frames)
res = calibrate.calibrate_layer("ffn.0", w0, L0.plan, L0.scale_normal64, L0.scale_outlier64, act,
                                [(t, f + 1) for f, t in enumerate(xs)], cw,
                                qb._lib.CalibConfig(iterations=3, batch_size=2))
os.environ["QARVD_K7_OZAKI"] = "0"
calibrate.calibrate_layer("ffn.0", w0, L0.plan, L0.scale_normal64, L0.scale_outlier64, act,
                          [(t, f + 1) for f, t in enumerate(xs)], cw, qb._lib.CalibConfig(iterations=2, batch_size=2))
os.environ.pop("QARVD_K7_OZAKI")
# K6: the Eq. 5 loss over bf16 samples
batch = [(t.to(torch.bfloat16), f + 1) for f, t in enumerate(xs)]
loss = calibrate.weighted_loss(batch, L0, w0, cw, act)
# K3 -> K5 -> K4 (percentile search) through the calibration shard
shard = calibrate.CalibrationShard([spec0, spec2], [0, 1], frames=frames, rows=rows)
shard.setup()
recs = shard.run()
torch.cuda.synchronize()
print("sanitize driver ok", float(res.final_loss), float(loss), len(recs))
