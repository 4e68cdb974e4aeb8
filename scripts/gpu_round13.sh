cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QARVD_GEMM_CG=1 QARVD_GEMM_BN=192 timeout 120 python scripts/gemm_trace.py ffn2 1536 8960 188 > gpurun_out/trace13_ffn2_192.txt 2>&1
QARVD_GEMM_CG=1 QARVD_GEMM_BN=192 QARVD_GEMM_DEBUG=2 timeout 120 python scripts/gemm_trace.py ffn2 1536 8960 188 > gpurun_out/trace13_ffn2_192_mma.txt 2>&1
QARVD_GEMM_CG=1 QARVD_GEMM_BN=128 timeout 120 python scripts/gemm_trace.py ffn0 8960 1536 32 > gpurun_out/trace13_ffn0_128.txt 2>&1
QARVD_GEMM_CG=2 QARVD_GEMM_BN=256 timeout 120 python scripts/gemm_trace.py ffn0 8960 1536 32 > gpurun_out/trace13_ffn0_256_2.txt 2>&1
echo done >> gpurun_out/status13.txt
