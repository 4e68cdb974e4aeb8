cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in 2 0; do
QARVD_GEMM_DEBUG=$d timeout 300 python scripts/gemm_trace.py ffn0 8960 1536 32 1 > gpurun_out/tr59_$d.log 2>&1
done
