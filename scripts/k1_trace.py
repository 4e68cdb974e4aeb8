import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_21072_b200 as qb
from paper_2605_21072_b200 import _lib, engine, synth
M = 4680
k = int(sys.argv[1])
plan = engine.build_plan("l", k, list(range(0, k, k // 32))[:32])
g = torch.from_numpy(plan.gather).cuda()
x = synth.synth_activation(M, k, seed=3)
xq = torch.empty((M, plan.k_pad), dtype=torch.int8, device="cuda")
sx = torch.empty(M, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.call("qarvd_quantize_act", x.data_ptr(), qb.BF16, M, k, k, g.data_ptr(), plan.k_pad, 0, 0.0, 8,
                      xq.data_ptr(), plan.k_pad, sx.data_ptr(), None, None, st)
f(); torch.cuda.synchronize()
os.environ["QARVD_K1_DEBUG"] = "2"
f(); torch.cuda.synchronize()
