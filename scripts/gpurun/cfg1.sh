cd /root/repo
for cfg in "256 2 2" "128 1 2" "128 1 1" "128 2 2" "256 1 2"; do set -- $cfg
echo "== BN=$1 CG=$2 KS=$3"; QARVD_GEMM_BN=$1 QARVD_GEMM_CG=$2 QARVD_GEMM_KS=$3 timeout 60 python scripts/cta_times.py 1536 1536 32 0 2>&1 | grep "start:" | head -1
done
