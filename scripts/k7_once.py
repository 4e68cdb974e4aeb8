"""A few K7 iterations at the Wan 1536x1536 shape (21 x 1560-token samples, batch 8), for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import calibrate, engine, synth
spec = synth.wan_registry(blocks=1)[0]
w = synth.synth_weight(spec, seed=1)
plan = engine.build_plan(spec.name, spec.in_dim, qb.analyze_layer(spec.name, w).aligned_outliers)
layer = engine.prepare_weights(spec.name, w, plan)
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
xs = [synth.synth_activation(rows, spec.in_dim, seed=3, frame=f).double() for f in range(frames)]
act = max(float(x.abs().max()) for x in xs) / 127.0
cw = calibrate.weighting_strategy("heuristic_exp", frames)
res = calibrate.calibrate_layer(spec.name, w, plan, layer.scale_normal64, layer.scale_outlier64, act,
                                [(x, f + 1) for f, x in enumerate(xs)], cw,
                                qb._lib.CalibConfig(iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 2, batch_size=8))
torch.cuda.synchronize()
print("ok", res.final_loss)
