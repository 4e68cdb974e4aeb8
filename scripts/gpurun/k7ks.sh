python - <<'PY'
import os, sys, json
sys.path.insert(0, '.')
import torch
import bench
for ks in ("auto", "2"):
    if ks != "auto": os.environ["QARVD_GEMM_KS"] = ks
    r = bench.adaround_bench(torch, iters=10)
    print("KS", ks, json.dumps({k: r[k] for k in ("ms_per_iteration", "fixed_ms", "final_loss")}))
PY
unset QARVD_GEMM_KS
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:dual_gemm' --csv --log-file gpurun_out/k7_gemm_launches.csv python scripts/k7_once.py 2 > /dev/null 2>&1; echo rc=$?
