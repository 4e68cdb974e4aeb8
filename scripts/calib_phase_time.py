"""Isolated device times of the calibration step's phases (300 Wan layers): K3 analyze, device
plan + K5, K4 search -- each timed alone after a warm-up run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_21072_b200 import _lib, calibrate, outlier, synth
from paper_2605_21072_b200.engine import _stream
specs = synth.wan_registry()
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
shard = calibrate.CalibrationShard(specs, list(range(len(specs))), frames, rows,
                                   frame_weights=calibrate.weighting_strategy("heuristic_exp", frames))
shard.setup()
shard.run(); shard.run()


def t(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


k3 = lambda: outlier.analyze_layers_async([s.name for s in shard.specs], shard.w, out=shard._rep)
k5 = lambda: _lib.call("qarvd_prepare_weights_planned", shard._jobs, len(shard.specs), 8, None, _stream())
def k4():
    for g, (jobs, nj, pct, nc, w, res) in enumerate(shard._k4):
        _lib.call("qarvd_scale_search_async", jobs, nj, pct, nc, w, 8, shard._flags[g:g + 1].data_ptr(), _stream())
print(f"K3 {t(k3):.3f} ms   K5 {t(k5):.3f} ms   K4 {t(k4):.3f} ms   step {t(shard.run):.3f} ms")
