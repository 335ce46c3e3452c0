"""Event-timed standalone full-p screening pass (k_screen_full) on a config's
design: algorithmic bytes / duration vs the measured HBM peak."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = synth.by_name(name)
X = gs.DesignMatrix(c.X)
n, p = c.X.shape
rng = np.random.default_rng(0)
center = c.y / np.max(np.abs(c.X.T @ c.y))
es = c.X.dtype.itemsize if not hasattr(c.X, "nnz") else 8
out = {}
for r in (0.0, 1e-3, 1e-1):
    ms = gs.PathTimer.screen_pass_ms(X, center, r, reps=reps)
    byts = n * p * es + 9 * p + 8 * n
    out[str(r)] = dict(ms=ms, gbs=byts / (ms * 1e-3) / 1e9)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
print(json.dumps(dict(config=name, n=n, p=p, peak_gbs=peak, runs=out)))
