cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu11.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status11.txt
timeout 600 python scripts/gemm_probe.py > gpurun_out/probe11.json 2> gpurun_out/probe11.err; echo "probe exit $?" >> gpurun_out/status11.txt
timeout 600 python scripts/bench_kernels.py > gpurun_out/kern11.json 2> gpurun_out/kern11.err; echo "kern exit $?" >> gpurun_out/status11.txt
