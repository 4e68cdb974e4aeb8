ncu --set full --clock-control none --import-source on -k regex:hist_kernel -c 1 -o gpurun_out/prof_hist -f python scripts/calib_once.py > gpurun_out/histprof.log 2>&1; echo rc=$?
