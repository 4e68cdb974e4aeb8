"""Timeline of one calibration step (CalibrationShard.run) with events on both streams."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_21072_b200 import calibrate, synth, outlier, engine

specs = synth.wan_registry()
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
w = calibrate.weighting_strategy("heuristic_exp", frames)
shard = calibrate.CalibrationShard(specs, list(range(len(specs))), frames, rows, frame_weights=w)
shard.setup()
for _ in range(2):
    shard.run()
torch.cuda.synchronize()
for rep in range(3):
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e0.record()
    recs = shard.run()
    e1 = torch.cuda.Event(enable_timing=True); e1.record()
    torch.cuda.synchronize()
    print(f"step {rep}: events {e0.elapsed_time(e1):.2f} ms, host wall {(time.perf_counter()-h0)*1e3:.2f} ms")
# phase breakdown with explicit syncs
def ph(name, fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"  {name:30s} {(time.perf_counter()-t)*1e3:8.2f} ms"); return r
dev_rep = ph("K3 analyze (async + sync)", lambda: outlier.analyze_layers_async([s.name for s in shard.specs], shard.w))
reps = ph("collect_reports", lambda: outlier.collect_reports(dev_rep))
plans = ph("build_plan x300 (host)", lambda: [engine.build_plan(s.name, s.in_dim, r.aligned_outliers) for s, r in zip(shard.specs, reps)])
layers = ph("K5 prepare_weights_batched", lambda: engine.prepare_weights_batched([s.name for s in shard.specs], shard.w, plans, check_finite=False))
groups = {}
for i, x in enumerate(shard.x):
    groups.setdefault(x.shape[0] // shard.frames, []).append(i)
def k4():
    out = []
    for r_, idx in groups.items():
        out.append(calibrate.scale_search_async([shard.x[i] for i in idx], shard.frames, shard.weights))
    return out
res = ph("K4 search (2 groups)", k4)
ph("results D2H", lambda: [r.cpu() for r in res])
