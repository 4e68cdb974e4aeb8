cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu21.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status21.txt
timeout 600 python scripts/bench_kernels.py > gpurun_out/kern21.json 2> gpurun_out/kern21.err; echo "kern exit $?" >> gpurun_out/status21.txt
