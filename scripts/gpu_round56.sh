cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t56.log 2>&1; echo "tests exit $?" >> gpurun_out/status56.txt
for i in 1 2; do
timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b56_$i.json 2> gpurun_out/b56_$i.err; echo "bench exit $?" >> gpurun_out/status56.txt
done
timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr56.log 2>&1
timeout 300 python scripts/gemm_trace.py ffn2 1536 8960 192 0 > gpurun_out/tr56_ffn2.log 2>&1
