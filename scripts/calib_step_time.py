"""Device time of the 300-layer calibration step (CalibrationShard.run), best of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_21072_b200 import calibrate, synth
specs = synth.wan_registry()
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
shard = calibrate.CalibrationShard(specs, list(range(len(specs))), frames, rows,
                                   frame_weights=calibrate.weighting_strategy("heuristic_exp", frames))
shard.setup()
for _ in range(2):
    shard.run()
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); shard.run(); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
print(os.environ.get("QARVD_CALIB_ORDER", "hist_first"), "step ms", min(ts), "layers/s", 300 / min(ts) * 1e3)
