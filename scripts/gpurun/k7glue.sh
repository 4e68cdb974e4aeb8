# full ncu capture of one K7 iteration's glue kernels (act codes, residual, D' slices)
ncu --set full --clock-control none --import-source on -k 'regex:act_codes_group|resid_kernel|d_slices_t' --launch-skip 6 --launch-count 3 \
    -o gpurun_out/prof_k7_glue python scripts/k7_once.py 1 > gpurun_out/k7_glue.log 2>&1; echo rc=$?
