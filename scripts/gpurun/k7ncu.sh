# full ncu capture of one K7 iteration's two slice GEMMs (GEMM1 = X^ What^T, GEMM2 = D'^T X^)
ncu --set full --clock-control none --import-source on -k 'regex:dual_gemm' --launch-skip 3 --launch-count 2 \
    -o gpurun_out/prof_k7_gemm python scripts/k7_once.py 1 > gpurun_out/k7_ncu_full.log 2>&1; echo rc=$?
