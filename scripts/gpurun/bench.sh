timeout 1200 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r2a.err
timeout 300 python bench.py --ffn-only --steps 5 --warmup 3 > gpurun_out/ffn_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dual_gemm -s 0 -c 2 -o gpurun_out/prof_k2_r2 -f python bench.py --ffn-only --steps 5 --warmup 3 > gpurun_out/ncu_k2.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_k2.log
