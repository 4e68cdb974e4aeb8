# ncu launch list (gpu__time_duration, cold, serialised) of the headline FFN bench command
cd /root/repo
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:dual_gemm|quant_act' -c 60 --csv --log-file gpurun_out/r2_ffn_launches.csv \
  python bench.py --ffn-only --steps 2 --warmup 3 > gpurun_out/r2_ffn_ncu.log 2>&1; echo rc=$?
python scripts/launch_summary.py gpurun_out/r2_ffn_launches.csv 2>&1 | head -12
