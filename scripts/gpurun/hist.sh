timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "k4 or search or percentile or calib or shard" 2>&1 | tail -2
timeout 120 python scripts/calib_phase_time.py 2>&1 | tail -1
timeout 120 python scripts/calib_step_time.py 2>&1 | tail -1
