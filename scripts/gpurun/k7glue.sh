# K7: parity tests, per-iteration timing and the launch list of 2 iterations
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "calibrate_layer or adaround or f64" 2>&1 | tail -2
timeout 300 ./tests/cpp/build/test_dropin 2>&1 | grep -E "DROPIN|FAIL" | tail -2
timeout 300 python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import torch, bench
for _ in range(2):
    r = bench.adaround_bench(torch, iters=20)
    print("K7", json.dumps({k: r[k] for k in ("ms_per_iteration", "final_loss")}))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:act_codes|resid|d_slices|weights_kernel|grad_kernel' --csv --log-file gpurun_out/k7glue_launches.csv python scripts/k7_once.py 2 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/k7glue_launches.csv 2>/dev/null | head -12
