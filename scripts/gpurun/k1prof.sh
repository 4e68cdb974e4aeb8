python bench.py --ffn-only --steps 5 --warmup 3 > gpurun_out/k1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:quant_act -s 0 -c 2 -o gpurun_out/prof_k1_r2 -f python bench.py --ffn-only --steps 5 --warmup 3 > gpurun_out/ncu_k1.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_k1.log
