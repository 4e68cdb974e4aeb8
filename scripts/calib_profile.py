"""Phase timing of one calibration step (config-4 shape, 300 layers, 1 GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_21072_b200 import calibrate, synth, outlier, engine

specs = synth.wan_registry()
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
w = calibrate.weighting_strategy("heuristic_exp", frames)
shard = calibrate.CalibrationShard(specs, list(range(len(specs))), frames, rows, frame_weights=w)
t0 = time.perf_counter(); shard.setup(); print(f"setup {time.perf_counter()-t0:.1f}s")
shard.run(); torch.cuda.synchronize()

def phase(name, fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"  {name:28s} {(time.perf_counter()-t)*1e3:8.2f} ms"); return r

for rep in range(2):
    print("step", rep)
    t_all = time.perf_counter()
    dev_rep = phase("K3 launch+run", lambda: outlier.analyze_layers_async([s.name for s in shard.specs], shard.w))
    groups = {}
    for i, x in enumerate(shard.x):
        groups.setdefault(x.shape[0] // shard.frames, []).append(i)
    def k4():
        out = {}
        for r_, idx in groups.items():
            res = calibrate.scale_search_async([shard.x[i] for i in idx], shard.frames, shard.weights)
            for j, i in enumerate(idx):
                out[i] = res[j]
        return out
    search = phase("K4 launch+run", k4)
    reps = phase("collect_reports (D2H)", lambda: outlier.collect_reports(dev_rep))
    def k5():
        L = []
        for spec, wt, rp in zip(shard.specs, shard.w, reps):
            plan = engine.build_plan(spec.name, spec.in_dim, rp.aligned_outliers)
            L.append(engine.prepare_weights(spec.name, wt, plan, check_finite=False))
        return L
    layers = phase("K5 per layer", k5)
    phase("per-layer D2H of results", lambda: [(search[i].cpu(), L.scale_outlier64.cpu(), L.scale_normal64.cpu()) for i, L in enumerate(layers)])
    print(f"  total {(time.perf_counter()-t_all)*1e3:.1f} ms")
