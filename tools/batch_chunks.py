"""Run cfg4 problems [lo, hi) as one batch; print which chunk fails (debug)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth
lo, hi = int(sys.argv[1]), int(sys.argv[2])
X0, y0, _ = synth.cfg4_shared()
rows = np.stack([synth.cfg4_rows(b) for b in range(lo, hi)]).astype(np.int32)
D0 = gs.DesignMatrix(X0)
bs = gs.BatchPathSolver(D0, y0, rows)
grids = np.stack([gs.lambda_grid(bs.lambda_max[b], 50, 2.0) for b in range(hi - lo)])
eps = min(1e-8 * float(y0[rows[b]] @ y0[rows[b]]) for b in range(hi - lo))
t = time.perf_counter()
res = bs.run_paths(grids, gs.SolverConfig(epsilon=eps, max_passes=100_000))
print(json.dumps(dict(lo=lo, hi=hi, s=time.perf_counter() - t, conv=int(res["converged"].sum()))))
