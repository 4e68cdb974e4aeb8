timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "k1 or quantize or chain or fold or stack or act or qarq or bulk or k5 or weights or calib or w4 or bits" > gpurun_out/k1check_tests.log 2>&1; tail -2 gpurun_out/k1check_tests.log
timeout 300 ./tests/cpp/build/test_dropin 2>&1 | grep -E "DROPIN|FAIL" | tail -2
bash scripts/gpurun/k1micro.sh 2>&1 | grep -E "product K1|differ"
timeout 300 python scripts/k1_flush_probe.py 2>&1 | grep "flush 2"
timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('FFN', round(d['ms_per_step']*1e3,1), 'us', d['value'], {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'}, 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"
