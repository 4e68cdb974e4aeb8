cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_ffn.py > gpurun_out/prof_plain39.log 2>&1; echo "plain exit $?" >> gpurun_out/status39.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quant_act -s 2 -c 2 -o gpurun_out/prof_k1_39 python scripts/prof_ffn.py > gpurun_out/ncu39.log 2>&1; echo "ncu exit $?" >> gpurun_out/status39.txt
