cd /root/repo
QARVD_K1_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1 or chain or fold or stack or act" 2>&1 | tail -2
for p in 0 1 0 1; do QARVD_K1_PERSIST=$p timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('persist=$p FFN', round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'})"; done
