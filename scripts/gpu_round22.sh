cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu22.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status22.txt
timeout 900 python bench.py > gpurun_out/bench22.json 2> gpurun_out/bench22.err; echo "bench exit $?" >> gpurun_out/status22.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench22_ref.json 2> gpurun_out/bench22_ref.err; echo "ref exit $?" >> gpurun_out/status22.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches22.csv python bench.py --steps 5 --warmup 3 --no-calib --no-cpu-baseline > gpurun_out/ncu22.log 2>&1; echo "ncu list exit $?" >> gpurun_out/status22.txt
