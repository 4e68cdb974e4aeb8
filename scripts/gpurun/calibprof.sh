ncu --set full --clock-control none --import-source on -k 'regex:column_norms|select_outliers|prep_weights_batched' -c 6 \
    -o gpurun_out/prof_calib_k35 -f python scripts/calib_once.py > gpurun_out/calibprof.log 2>&1; echo rc=$?
