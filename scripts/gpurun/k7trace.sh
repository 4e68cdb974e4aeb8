QARVD_GEMM_TRACE=1 QARVD_GEMM_TRACE_CTA=10 python scripts/k7_once.py 1 > gpurun_out/k7_trace.log 2>&1; echo rc=$?
