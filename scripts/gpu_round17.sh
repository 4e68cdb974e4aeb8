cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "2 256 2" "2 256 1" "1 192 1" "1 256 1" "2 128 2" "1 128 1"; do set -- $cfg; QARVD_GEMM_CG=$1 QARVD_GEMM_BN=$2 QARVD_GEMM_KS=$3 timeout 300 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q -x -k "k2 or linear" > gpurun_out/t_gpu17_$1_$2_$3.log 2>&1; echo "cfg $1 $2 $3 exit $?" >> gpurun_out/status17.txt; done
timeout 600 python scripts/gemm_probe.py > gpurun_out/probe17.json 2> gpurun_out/probe17.err; echo "probe exit $?" >> gpurun_out/status17.txt
QARVD_GEMM_CG=2 QARVD_GEMM_BN=256 QARVD_GEMM_KS=2 timeout 120 python scripts/gemm_trace.py ffn0 8960 1536 32 > gpurun_out/trace17_ffn0.txt 2>&1
