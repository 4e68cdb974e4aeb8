cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest -p no:cacheprovider tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/status2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke exit $?" >> gpurun_out/status2.txt
timeout 600 python bench.py > gpurun_out/bench2.log 2>&1; echo "bench exit $?" >> gpurun_out/status2.txt
timeout 300 python scripts/prof_ffn.py > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv python scripts/prof_ffn.py > gpurun_out/ncu_l.log 2>&1; echo "ncu list exit $?" >> gpurun_out/status2.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dual_gemm -s 2 -c 2 -o gpurun_out/prof_gemm2 python scripts/prof_ffn.py > gpurun_out/ncu_f.log 2>&1; echo "ncu full exit $?" >> gpurun_out/status2.txt
