cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/epi_rate.bin > gpurun_out/epi_rate52.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t52.log 2>&1; echo "tests exit $?" >> gpurun_out/status52.txt
for i in 1 2; do
timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b52_$i.json 2> gpurun_out/b52_$i.err; echo "bench exit $?" >> gpurun_out/status52.txt
done
timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr52.log 2>&1
