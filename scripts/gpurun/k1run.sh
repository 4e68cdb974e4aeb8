cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1 or quantize or chain or fold or stack or act or qarq or bulk or k5 or bits or fused or linear_handle" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FFN', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'})"; done
