"""ffn.0 K2 timing under tile-config overrides (QARVD_GEMM_BN / _CG / _KS)."""
import os, sys, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = open(os.path.join(ROOT, "scripts", "epi_probe.py")).read().split("code = r'''")[1].split("''' % ROOT")[0] % ROOT
for cfg in [("256", "2", "2"), ("128", "2", "2"), ("128", "2", "1"), ("192", "2", "1"), ("256", "1", "2")]:
    env = dict(os.environ, QARVD_GEMM_BN=cfg[0], QARVD_GEMM_CG=cfg[1], QARVD_GEMM_KS=cfg[2])
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print("BN/CG/KS", "/".join(cfg), r.stdout.strip() or r.stderr[-300:], flush=True)
