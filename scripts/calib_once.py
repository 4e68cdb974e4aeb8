"""One calibration step (300 layers) for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_21072_b200 import calibrate, synth
specs = synth.wan_registry()
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
shard = calibrate.CalibrationShard(specs, list(range(len(specs))), frames, rows,
                                   frame_weights=calibrate.weighting_strategy("heuristic_exp", frames))
shard.setup()
torch.cuda.synchronize()
shard.run()
torch.cuda.synchronize()
print("ok")
