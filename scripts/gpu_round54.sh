cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in 0 16; do
QARVD_GEMM_DEBUG=$d timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr54_$d.log 2>&1
done
QARVD_GEMM_DEBUG=1 timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr54_1.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t54.log 2>&1; echo "tests exit $?" >> gpurun_out/status54.txt
for i in 1 2; do
timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b54_$i.json 2> gpurun_out/b54_$i.err; echo "bench exit $?" >> gpurun_out/status54.txt
done
