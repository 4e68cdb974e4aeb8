for cfg in "" "QARVD_GEMM_CG=1" "QARVD_GEMM_CG=1 QARVD_GEMM_BN=128" "QARVD_GEMM_CG=1 QARVD_GEMM_KS=1"; do
  env $cfg timeout 300 python bench.py --ffn-only --steps 300 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$cfg]', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'})"
done
