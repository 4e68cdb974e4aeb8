cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_ffn.py > gpurun_out/s2k_plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_act -s 2 -c 1 -o gpurun_out/s2_prof_k1x python scripts/prof_ffn.py > gpurun_out/s2k_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/s2k_status.txt
