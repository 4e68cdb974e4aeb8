ncu --set full --clock-control none --import-source on -k regex:quant_act_bulk -s 100 -c 1 -o gpurun_out/prof_k1bulk_u -f python scripts/k1_flush_probe.py > gpurun_out/k1b2.log 2>&1; echo rc=$?
