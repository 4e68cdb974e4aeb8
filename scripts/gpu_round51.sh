cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t51.log 2>&1; echo "tests exit $?" >> gpurun_out/status51.txt
for i in 1 2; do
timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b51_reg$i.json 2> gpurun_out/b51_reg$i.err; echo "bench reg exit $?" >> gpurun_out/status51.txt
QARVD_GEMM_EPIREG=0 timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b51_old$i.json 2> gpurun_out/b51_old$i.err; echo "bench old exit $?" >> gpurun_out/status51.txt
done
timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr51_reg.log 2>&1
QARVD_GEMM_EPIREG=0 timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr51_old.log 2>&1
timeout 300 python scripts/gemm_trace.py ffn2 1536 8960 192 0 > gpurun_out/tr51_ffn2.log 2>&1
