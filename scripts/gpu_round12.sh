cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu12.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status12.txt
for cfg in "1 192" "2 192" "1 256" "2 128"; do set -- $cfg; QARVD_GEMM_CG=$1 QARVD_GEMM_BN=$2 timeout 300 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q -x -k "k2 or linear" > gpurun_out/t_gpu12_$1_$2.log 2>&1; echo "cfg $1 $2 exit $?" >> gpurun_out/status12.txt; done
timeout 600 python scripts/gemm_probe.py > gpurun_out/probe12.json 2> gpurun_out/probe12.err; echo "probe exit $?" >> gpurun_out/status12.txt
