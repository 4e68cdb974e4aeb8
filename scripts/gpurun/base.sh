set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_base_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2_base_tests.log
timeout 900 python bench.py > gpurun_out/r2_base_bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/r2_base_bench.log
