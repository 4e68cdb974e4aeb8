grep -o -w 'fma\|avx2' /proc/cpuinfo | sort | uniq -c; grep -m1 "model name" /proc/cpuinfo; nproc
timeout 900 ./tests/cpp/build/test_dropin > gpurun_out/dropin.log 2>&1; echo "dropin rc=$?"
tail -32 gpurun_out/dropin.log
timeout 600 ./tests/cpp/build/test_no_ref_compute > gpurun_out/noref.log 2>&1; echo "noref rc=$?"
tail -3 gpurun_out/noref.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/gputests.log
timeout 300 python -m pytest tests/test_crmath.py -q 2>&1 | tail -2
