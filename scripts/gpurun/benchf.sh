cd /root/repo
timeout 1200 python bench.py > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_r2f.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_r2f_ref.json 2>&1; echo "ref rc=$?"
timeout 600 python scripts/stack_breakdown.py 10 > gpurun_out/stack_breakdown.md 2>/dev/null; echo "stack rc=$?"
