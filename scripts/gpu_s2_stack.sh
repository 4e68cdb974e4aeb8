cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "stack or chain" > gpurun_out/s2s_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2s_status.txt
timeout 900 python bench.py --steps 200 --no-cpu-baseline --no-calib > gpurun_out/s2s_bench.json 2> gpurun_out/s2s_bench.err; echo "bench exit $?" >> gpurun_out/s2s_status.txt
