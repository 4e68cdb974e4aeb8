cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_ffn.py > gpurun_out/prof_plain58.log 2>&1; echo "plain exit $?" >> gpurun_out/status58.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dual_gemm -s 2 -c 2 -o gpurun_out/prof_gemm_58 python scripts/prof_ffn.py > gpurun_out/ncu58g.log 2>&1; echo "ncu gemm exit $?" >> gpurun_out/status58.txt
