"""Event-timed standalone full-p screening pass (k_screen_full) on a config's
design: algorithmic bytes / duration vs the measured HBM peak.
    python tools/time_screen.py cfg1|cfg2|cfg3 [reps] [p]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kw = {"p": int(sys.argv[3])} if len(sys.argv) > 3 else {}
c = synth.by_name(name, **kw)
X = gs.DesignMatrix(c.X)
n, p = c.X.shape
sparse = hasattr(c.X, "nnz") and not isinstance(c.X, np.ndarray)
if sparse:
    lmax = float(np.max(np.abs(c.X.T @ c.y)))
    byts = int(c.X.nnz) * 12 + 8 * (p + 1) + 9 * p + 8 * n      # data + row indices, column pointers, norms + marks, centre
else:
    lmax = float(np.max(np.abs(c.y @ c.X.astype(np.float64, copy=False)))) if p <= 200_000 else gs.DeviceSolver(X, c.y).lambda_max
    byts = n * p * c.X.dtype.itemsize + 9 * p + 8 * n
center = c.y / lmax
out = {}
for r in (0.0, 1e-3, 1e-1):
    ms = gs.PathTimer.screen_pass_ms(X, center, r, reps=reps)
    out[str(r)] = dict(ms=ms, gbs=byts / (ms * 1e-3) / 1e9)
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6650.0
for v in out.values():
    v["frac"] = v["gbs"] / peak
print(json.dumps(dict(config=name, n=n, p=p, bytes=byts, peak_gbs=peak, runs=out)))
