for cfg in "" "QARVD_K1_REG=2" "" "QARVD_K1_REG=2"; do
  env $cfg timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$cfg]', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'}, 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"
done
for cfg in "" "QARVD_K1_REG=2"; do env $cfg timeout 300 python scripts/k1_flush_probe.py 2>&1 | grep "gathered" | sed "s/^/[$cfg] /"; done
