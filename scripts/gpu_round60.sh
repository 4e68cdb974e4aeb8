cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench60.json 2> gpurun_out/bench60.err; echo "bench exit $?" >> gpurun_out/status60.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench60_ref.json 2> gpurun_out/bench60_ref.err; echo "ref exit $?" >> gpurun_out/status60.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches60.csv python bench.py --steps 5 --warmup 3 --no-calib --no-cpu-baseline > gpurun_out/ncu60.log 2>&1; echo "ncu list exit $?" >> gpurun_out/status60.txt
timeout 300 python scripts/prof_ffn.py > gpurun_out/prof_plain60.log 2>&1; echo "plain exit $?" >> gpurun_out/status60.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dual_gemm -s 2 -c 2 -o gpurun_out/prof_gemm_60 python scripts/prof_ffn.py > gpurun_out/ncu60g.log 2>&1; echo "ncu gemm exit $?" >> gpurun_out/status60.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_act -s 2 -c 2 -o gpurun_out/prof_k1_60 python scripts/prof_ffn.py > gpurun_out/ncu60k.log 2>&1; echo "ncu k1 exit $?" >> gpurun_out/status60.txt
