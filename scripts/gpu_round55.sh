cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sp in 0 1; do
QARVD_GEMM_SPIN=$sp timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr55_$sp.log 2>&1
QARVD_GEMM_SPIN=$sp timeout 300 python scripts/gemm_trace.py ffn2 1536 8960 192 0 > gpurun_out/tr55_ffn2_$sp.log 2>&1
QARVD_GEMM_SPIN=$sp timeout 300 python bench.py --no-calib --no-cpu-baseline > gpurun_out/b55_$sp.json 2> gpurun_out/b55_$sp.err
done
