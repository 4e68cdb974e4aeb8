timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/r2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke.log
timeout 1200 python bench.py > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_r2i.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_r2i_ref.json 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_r2i_ref.json
timeout 600 python scripts/stack_breakdown.py 10 > gpurun_out/stack_breakdown.md 2>/dev/null; echo "stack rc=$?"
timeout 300 ./tests/cpp/build/test_dropin > gpurun_out/dropin.log 2>&1; echo "dropin rc=$?"; grep -E "DROPIN|FAIL" gpurun_out/dropin.log | tail -2
