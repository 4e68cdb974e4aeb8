cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QARVD_GEMM_CG=2 timeout 300 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q -x -k "k2 or linear or smoke" > gpurun_out/t_cg2.log 2>&1; echo "cg2 tests exit $?" >> gpurun_out/status6.txt
QARVD_GEMM_CG=2 QARVD_GEMM_BN=256 timeout 300 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q -x -k "k2" > gpurun_out/t_cg2b.log 2>&1; echo "cg2 bn256 tests exit $?" >> gpurun_out/status6.txt
QARVD_GEMM_CG=1 timeout 300 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q -x -k "k2" > gpurun_out/t_cg1.log 2>&1; echo "cg1 tests exit $?" >> gpurun_out/status6.txt
timeout 600 python scripts/bench_kernels.py > gpurun_out/kern6.json 2> gpurun_out/kern6.err; echo "kern exit $?" >> gpurun_out/status6.txt
