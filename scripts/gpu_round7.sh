cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/gemm_probe.py > gpurun_out/probe7.json 2> gpurun_out/probe7.err; echo "probe exit $?" >> gpurun_out/status7.txt
timeout 900 python -m pytest -p no:cacheprovider tests/test_gpu_dropin.py -q -x -s > gpurun_out/t_dropin7.log 2>&1; echo "dropin exit $?" >> gpurun_out/status7.txt
