bash scripts/gpurun/k7.sh
bash scripts/gpurun/k7ncu.sh
