cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QARVD_K1_DEBUG=1 timeout 300 python scripts/prof_ffn.py > gpurun_out/prof_plain43.log 2>&1; echo "plain exit $?" >> gpurun_out/status43.txt
QARVD_K1_DEBUG=1 timeout 900 ncu --set full --clock-control none -k regex:quant_act -s 2 -c 2 -o gpurun_out/prof_k1_43 python scripts/prof_ffn.py > gpurun_out/ncu43.log 2>&1; echo "ncu exit $?" >> gpurun_out/status43.txt
