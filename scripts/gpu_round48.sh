cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "k2 or chain or gemm or linear" > gpurun_out/t48a.log 2>&1; echo "tests tma exit $?" >> gpurun_out/status48.txt
QARVD_GEMM_DIRECT=1 timeout 600 python -m pytest tests -m gpu -x -q -k "k2 or chain or gemm or linear" > gpurun_out/t48b.log 2>&1; echo "tests direct exit $?" >> gpurun_out/status48.txt
for i in 1 2; do
timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b48_tma$i.json 2> gpurun_out/b48_tma$i.err; echo "bench tma exit $?" >> gpurun_out/status48.txt
QARVD_GEMM_DIRECT=1 timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b48_dir$i.json 2> gpurun_out/b48_dir$i.err; echo "bench direct exit $?" >> gpurun_out/status48.txt
done
timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr48_tma.log 2>&1
QARVD_GEMM_DIRECT=1 timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr48_dir.log 2>&1
