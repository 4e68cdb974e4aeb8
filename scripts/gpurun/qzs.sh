cd /root/repo
for dbg in 0; do for fq in 0 1; do
QARVD_GEMM_DEBUG=$dbg QARVD_BENCH_STATIC=1 QARVD_FUSE_QUANT=$fq timeout 300 python bench.py --ffn-only --steps 300 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dbg=$dbg static FQ=$fq FFN', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'})"
done; done
