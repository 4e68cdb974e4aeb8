cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu28.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status28.txt
timeout 900 python bench.py --no-calib --steps 500 > gpurun_out/bench28.json 2> gpurun_out/bench28.err; echo "bench exit $?" >> gpurun_out/status28.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches28.csv python bench.py --steps 5 --warmup 3 --no-calib --no-cpu-baseline > gpurun_out/ncu28.log 2>&1; echo "ncu list exit $?" >> gpurun_out/status28.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_act -s 2 -c 2 -o gpurun_out/prof_k1_28 python scripts/prof_ffn.py > gpurun_out/ncu28b.log 2>&1; echo "ncu full exit $?" >> gpurun_out/status28.txt
