cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu9.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status9.txt
QARVD_GEMM_CG=1 timeout 300 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q -x -k "k2 or linear" > gpurun_out/t_gpu9_cg1.log 2>&1; echo "cg1 tests exit $?" >> gpurun_out/status9.txt
timeout 600 python scripts/gemm_probe.py > gpurun_out/probe9.json 2> gpurun_out/probe9.err; echo "probe exit $?" >> gpurun_out/status9.txt
