QARVD_K1_REG=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1 or quantize or chain or fold or stack or act or qarq" > gpurun_out/k1g_tests.log 2>&1; tail -1 gpurun_out/k1g_tests.log
for cfg in "" "QARVD_K1_REG=2"; do env $cfg timeout 300 python scripts/k1_flush_probe.py 2>&1 | grep "gathered): flush 2" | sed "s/^/[$cfg] /"; done
for cfg in "" "QARVD_K1_REG=2"; do
  env $cfg timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$cfg]', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'})"
done
