timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -x -k "k1 or quantize or chain or fold or stack or act or qarq or bulk or dropin" > gpurun_out/k1p2_tests.log 2>&1; tail -1 gpurun_out/k1p2_tests.log
bash scripts/gpurun/k1micro.sh 2>&1 | grep -E "product K1|differ"
timeout 300 python scripts/k1_flush_probe.py 2>&1 | grep "flush 2"
timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FFN', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'}, 'launches', d['gpu_launches'])"
