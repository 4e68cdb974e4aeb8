for v in 1 0; do echo "QARVD_K1_BULK=$v"; QARVD_K1_BULK=$v python scripts/k1_flush_probe.py 2>&1 | tail -6; done
