cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/s2_status.txt
timeout 900 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo "bench exit $?" >> gpurun_out/s2_status.txt
