python scripts/calib_once.py > gpurun_out/calib_plain.log 2>&1 && \
timeout 800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:^(?!.*(synth|scale_cols)).*' --csv --log-file gpurun_out/calib_launches.csv python scripts/calib_once.py > gpurun_out/calib_ncu.log 2>&1; echo rc=$?
