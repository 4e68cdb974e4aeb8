# fused consumer-K1 GEMM: parity tests, then FFN step A/B (unfused vs fused, per-token and static)
cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_quant or chain_fold or k2_tile or k2_acc" > gpurun_out/qz_tests.log 2>&1; tail -3 gpurun_out/qz_tests.log
for st in 0 1; do for fq in 0 1 0 1; do
QARVD_BENCH_STATIC=$st QARVD_FUSE_QUANT=$fq timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>gpurun_out/qz_bench_$fq.err | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('static=$st FQ=$fq FFN', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'})"
done; done
