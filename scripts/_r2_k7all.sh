bash scripts/_r2_k7.sh
bash scripts/_r2_k7ncu.sh
