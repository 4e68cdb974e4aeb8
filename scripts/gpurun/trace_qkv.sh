for cfg in "2 256 2" "1 128 2" "1 128 1"; do
  set -- $cfg
  QARVD_GEMM_CG=$1 QARVD_GEMM_BN=$2 QARVD_GEMM_KS=$3 python scripts/gemm_trace.py qkv 1536 1536 32 2>&1 | grep -v "^$" | head -12
  QARVD_GEMM_TRACE_CTA=140 QARVD_GEMM_CG=$1 QARVD_GEMM_BN=$2 QARVD_GEMM_KS=$3 python scripts/gemm_trace.py qkv 1536 1536 32 2>&1 | grep -v "^$" | sed -n 2,8p
done
