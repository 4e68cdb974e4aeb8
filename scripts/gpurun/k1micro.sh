python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2605_21072_b200 import synth
x = synth.synth_activation(4680, 1536, seed=3)
x.view(__import__('torch').int16).cpu().numpy().tofile('/tmp/x_real.bin')
PY
./scripts/micro/k1_micro /tmp/x_real.bin
