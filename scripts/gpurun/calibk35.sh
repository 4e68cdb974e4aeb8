python -m pytest tests/test_gpu_parity.py -q -x -k "k5 or k3 or outlier or analyze or calib or plan or prep or weights" 2>&1 | tail -2
python scripts/calib_step_time.py 2>&1 | tail -1
bash scripts/gpurun/calib.sh
