python -m pytest tests/test_gpu_parity.py -q -x -k "k1 or quantize or chain or fold or stack or smoke or act" 2>&1 | tail -3
for v in 1 0; do
  QARVD_K1_BULK=$v python bench.py --ffn-only --steps 300 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('K1_BULK=$v', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'}, d['quantize_roofline']['achieved_x'], d['quantize_roofline']['achieved_u'])"
done
