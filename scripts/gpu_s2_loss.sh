cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "weighted_loss" > gpurun_out/s2l_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2l_status.txt
