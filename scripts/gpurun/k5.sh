timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "k5 or prep or weights or calib or shard or w4 or W4 or bits or qarq or stack or chain" > gpurun_out/k5_tests.log 2>&1; tail -2 gpurun_out/k5_tests.log
timeout 300 ./tests/cpp/build/test_dropin 2>&1 | grep -E "DROPIN|FAIL" | tail -2
timeout 120 python scripts/calib_phase_time.py 2>&1 | tail -1
timeout 120 python scripts/calib_step_time.py 2>&1 | tail -1
timeout 300 bash scripts/gpurun/calib.sh
