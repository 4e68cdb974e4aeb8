cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_ffn.py > gpurun_out/prof_plain46.log 2>&1; echo "plain exit $?" >> gpurun_out/status46.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dual_gemm -s 2 -c 2 -o gpurun_out/prof_gemm_46 python scripts/prof_ffn.py > gpurun_out/ncu46.log 2>&1; echo "ncu exit $?" >> gpurun_out/status46.txt
