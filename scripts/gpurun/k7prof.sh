python scripts/k7_once.py 2 > gpurun_out/k7_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*(synth|scale_cols)).*' --csv --log-file gpurun_out/k7_launches.csv python scripts/k7_once.py 2 > gpurun_out/k7_ncu.log 2>&1; echo rc=$?
