cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu5.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status5.txt
timeout 600 python scripts/bench_kernels.py > gpurun_out/kern5.json 2> gpurun_out/kern5.err; echo "kern exit $?" >> gpurun_out/status5.txt
timeout 600 python bench.py > gpurun_out/bench5.log 2>&1; echo "bench exit $?" >> gpurun_out/status5.txt
