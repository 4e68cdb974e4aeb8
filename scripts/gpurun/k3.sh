timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k3 or outlier or analyze or detect or align or mad or median or calib or shard or k5" 2>&1 | tail -2
timeout 300 ./tests/cpp/build/test_dropin 2>&1 | grep -E "DROPIN|FAIL" | tail -2
timeout 120 python scripts/calib_phase_time.py 2>&1 | tail -1
timeout 120 python scripts/calib_step_time.py 2>&1 | tail -1
timeout 300 bash scripts/gpurun/calib.sh
