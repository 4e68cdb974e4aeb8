cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench23.json 2> gpurun_out/bench23.err; echo "bench exit $?" >> gpurun_out/status23.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches23.csv python bench.py --steps 5 --warmup 3 --no-calib --no-cpu-baseline > gpurun_out/ncu23.log 2>&1; echo "ncu list exit $?" >> gpurun_out/status23.txt
