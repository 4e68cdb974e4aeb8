cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 300 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -x -q -k "k1" > gpurun_out/t_k1.log 2>&1; echo "k1 exit $?" >> gpurun_out/status.txt
timeout 180 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -x -q -k "k2_acc and 77" > gpurun_out/t_k2a.log 2>&1; echo "k2a exit $?" >> gpurun_out/status.txt
timeout 900 python -m pytest -p no:cacheprovider tests/test_gpu_parity.py -q > gpurun_out/t_all.log 2>&1; echo "all exit $?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/status.txt
