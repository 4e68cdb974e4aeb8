"""Short FFN run for profiling (ncu launch lists / --set full): 3 eager chain launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_21072_b200 as qb  # noqa: E402
from paper_2605_21072_b200 import synth  # noqa: E402
from paper_2605_21072_b200.pipeline import QuantizedChain  # noqa: E402

layers = bench.build_ffn_layers(torch)
chain = QuantizedChain([layers[0][2], layers[1][2]], bench.M_TOKENS, epilogues=[qb.EPI_GELU, qb.EPI_NONE])
chain.x.copy_(synth.synth_activation(bench.M_TOKENS, bench.DIM, seed=7))
for _ in range(3):
    chain.launch()
torch.cuda.synchronize()
print("ok", qb._lib.launch_count())
