cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QARVD_GEMM_CG=2 QARVD_GEMM_BN=256 QARVD_GEMM_KS=2 timeout 120 python scripts/gemm_trace.py ffn0 8960 1536 32 > gpurun_out/trace18_ffn0_256.txt 2>&1
QARVD_GEMM_CG=1 QARVD_GEMM_BN=128 QARVD_GEMM_KS=2 timeout 120 python scripts/gemm_trace.py ffn0 8960 1536 32 > gpurun_out/trace18_ffn0_128.txt 2>&1
QARVD_GEMM_CG=2 QARVD_GEMM_BN=256 QARVD_GEMM_KS=2 timeout 120 python scripts/gemm_trace.py ffn2 1536 8960 188 > gpurun_out/trace18_ffn2_256.txt 2>&1
QARVD_GEMM_CG=2 QARVD_GEMM_BN=256 QARVD_GEMM_KS=2 QARVD_GEMM_DEBUG=2 timeout 120 python scripts/gemm_trace.py ffn0 8960 1536 32 > gpurun_out/trace18_ffn0_256_mma.txt 2>&1
