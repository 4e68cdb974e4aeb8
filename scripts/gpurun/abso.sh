# A/B of library builds on the FFN step (QARVD_B200_LIB)
cd /root/repo
for rep in 1 2; do for v in head ew8; do
QARVD_B200_LIB=paper_2605_21072_b200/libqarvd_$v.so timeout 300 python bench.py --ffn-only --steps 500 --warmup 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), {k: round(v*1e3,1) for k,v in d['kernel_ms'].items() if k!='note'})"
done; done
