cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x -k nothing_to_run > gpurun_out/t_gpu41.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status41.txt
timeout 900 python bench.py --no-calib --steps 500 > gpurun_out/bench41.json 2> gpurun_out/bench41.err; echo "bench exit $?" >> gpurun_out/status41.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches41.csv python bench.py --steps 5 --warmup 3 --no-calib --no-cpu-baseline > gpurun_out/ncu41.log 2>&1; echo "ncu list exit $?" >> gpurun_out/status41.txt
