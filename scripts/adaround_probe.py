"""K7 launch-list probe: calibrate_layer at the bench's Wan 1536 -> 1536 shape (21 x 1560-token
samples, batch 8) for QARVD_ADR_ITERS iterations (default 2); run under ncu for per-kernel times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

it = int(os.environ.get("QARVD_ADR_ITERS", "2"))
print(bench.adaround_bench(torch, iters=it))
