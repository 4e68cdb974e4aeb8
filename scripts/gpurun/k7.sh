python -m pytest tests/test_gpu_parity.py -q -x -k "calibrate_layer or adaround or f64" 2>&1 | tail -5
timeout 600 ./tests/cpp/build/test_dropin 2>&1 | grep -E "calibrate_|FAIL|DROPIN"
python - <<'PY'
import os, sys, json
sys.path.insert(0, '.')
import torch
import bench
for oz, bn in (("1", "128"), ("1", "256"), ("0", "128")):
    os.environ["QARVD_K7_OZAKI"] = oz
    os.environ["QARVD_F64_BN"] = bn
    r = bench.adaround_bench(torch, iters=10)
    print("OZAKI", oz, "BN", bn, json.dumps({k: r[k] for k in ("ms_per_iteration", "fixed_ms", "final_loss", "initial_loss")}))
PY
unset QARVD_K7_OZAKI QARVD_F64_BN
bash scripts/gpurun/k7prof.sh
