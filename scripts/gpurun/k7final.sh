python - <<'PY' > gpurun_out/k7_final_timing.txt 2>&1
import os, sys, json
sys.path.insert(0, '.')
import torch
import bench
for oz in ("1", "0", "1"):
    os.environ["QARVD_K7_OZAKI"] = oz
    r = bench.adaround_bench(torch, iters=20)
    print("OZAKI", oz, json.dumps({k: r[k] for k in ("ms_per_iteration", "fixed_ms", "final_loss", "initial_loss")}))
PY
cat gpurun_out/k7_final_timing.txt
bash scripts/gpurun/k7prof.sh
bash scripts/gpurun/k7ncu.sh
