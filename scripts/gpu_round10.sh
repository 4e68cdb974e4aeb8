cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest -p no:cacheprovider tests/test_gpu_dropin.py -q -x -s > gpurun_out/t_dropin10.log 2>&1; echo "dropin exit $?" >> gpurun_out/status10.txt
export QARVD_GEMM_CG=1
timeout 300 python scripts/prof_ffn.py > gpurun_out/prof_plain10.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dual_gemm -s 2 -c 2 -o gpurun_out/prof_gemm10 python scripts/prof_ffn.py > gpurun_out/ncu10.log 2>&1; echo "ncu exit $?" >> gpurun_out/status10.txt
