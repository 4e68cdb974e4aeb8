"""Calibration step time (300 Wan layers, one shard) under launch-order / K4-grid settings:
QARVD_CALIB_ORDER x QARVD_K4_SMS, median of 5 steps each, same shard."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_21072_b200 import calibrate, synth
specs = synth.wan_registry()
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
shard = calibrate.CalibrationShard(specs, list(range(len(specs))), frames, rows,
                                   frame_weights=calibrate.weighting_strategy("heuristic_exp", frames))
shard.setup()
torch.cuda.synchronize()
shard.run(); torch.cuda.synchronize()
for order in ("k3_first", "hist_first"):
    for sms in (148, 136, 128, 120, 112):
        os.environ["QARVD_CALIB_ORDER"] = order
        os.environ["QARVD_K4_SMS"] = str(sms)
        ts = []
        for _ in range(5):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            shard.run(); torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        ms = float(np.median(ts))
        print(f"{order:10s} K4 on {sms:3d} SMs: {ms:6.2f} ms per 300-layer step = {300 / ms * 1e3:7.0f} layers/s")
