"""cProfile of CalibrationShard.run() (config-4 shape, 300 layers, 1 GPU)."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_21072_b200 import calibrate, synth
specs = synth.wan_registry()
frames, rows = synth.WAN_FRAMES, synth.WAN_TOKENS_PER_FRAME
shard = calibrate.CalibrationShard(specs, list(range(len(specs))), frames, rows,
                                   frame_weights=calibrate.weighting_strategy("heuristic_exp", frames))
shard.setup()
for _ in range(2):
    shard.run()
torch.cuda.synchronize()
t = time.perf_counter(); shard.run(); torch.cuda.synchronize(); print(f"run {1e3*(time.perf_counter()-t):.1f} ms")
pr = cProfile.Profile(); pr.enable(); shard.run(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
