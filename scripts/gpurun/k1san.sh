python -m pytest tests/test_gpu_parity.py -q -x -k "bulk" 2>&1 | tail -2
bash scripts/gpurun/sanitize.sh
