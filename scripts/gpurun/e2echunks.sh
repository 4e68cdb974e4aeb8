for cfg in "" "QARVD_HOST_CHUNK_ROWS=384,1024,1024,1024" "QARVD_HOST_CHUNK_ROWS=256,768,1024,1024,1024" "QARVD_HOST_CHUNK_ROWS=512,1024,1280,1280" "QARVD_HOST_CHUNK_ROWS=256,512,1024,1024,1024,512" "QARVD_HOST_CHUNKS=6" "QARVD_HOST_CHUNK_ROWS=384,768,768,768,768,768"; do
  env $cfg timeout 300 python bench.py --ffn-only --steps 300 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$cfg]', 'step', round(d['ms_per_step']*1e3,1), 'us  e2e', round(d['e2e']['ms_per_step']*1e3,1), 'us', round(d['e2e']['value'],1))"
done
