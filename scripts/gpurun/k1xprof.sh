ncu --set full --clock-control none --import-source on -k regex:quant_act -s 95 -c 1 -o gpurun_out/prof_k1x_plain -f python scripts/k1_flush_probe.py > gpurun_out/k1xprof.log 2>&1; echo rc=$?
