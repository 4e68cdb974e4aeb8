cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q -x -k "k2 or linear" > gpurun_out/t_gpu14.log 2>&1; echo "k2 tests exit $?" >> gpurun_out/status14.txt
QARVD_GEMM_CG=1 QARVD_GEMM_BN=192 timeout 120 python scripts/gemm_trace.py ffn2 1536 8960 188 > gpurun_out/trace14_ffn2_192.txt 2>&1
QARVD_GEMM_CG=1 QARVD_GEMM_BN=128 timeout 120 python scripts/gemm_trace.py ffn0 8960 1536 32 > gpurun_out/trace14_ffn0_128.txt 2>&1
timeout 600 python scripts/gemm_probe.py > gpurun_out/probe14.json 2> gpurun_out/probe14.err; echo "probe exit $?" >> gpurun_out/status14.txt
