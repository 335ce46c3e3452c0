"""Time BASELINE configs[4] on one GPU: B bootstrap problems (n=500 rows drawn
with replacement from a shared 1000 x 50000 AR(1) design), each a 50-lambda
path to lambda_max/1e2, gap tolerance 1e-8 ||y_b||^2 per problem."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
p = int(sys.argv[2]) if len(sys.argv) > 2 else 50_000
T = 50
t0 = time.perf_counter()
X0, y0, _ = synth.cfg4_shared(p=p)
rows = np.stack([synth.cfg4_rows(b) for b in range(B)]).astype(np.int32)
t1 = time.perf_counter()
D0 = gs.DesignMatrix(X0)
bs = gs.BatchPathSolver(D0, y0, rows)
t2 = time.perf_counter()
grids = np.stack([gs.lambda_grid(bs.lambda_max[b], T, 2.0) for b in range(B)])
eps = np.array([1e-8 * float(y0[rows[b]] @ y0[rows[b]]) for b in range(B)])
res = bs.run_paths(grids, gs.SolverConfig(epsilon=1.0, max_passes=100_000), epsilons=eps)
t3 = time.perf_counter()
print(json.dumps(dict(config="cfg4", B=B, p=p, T=T, gen_s=t1 - t0, setup_s=t2 - t1, run_s=t3 - t2,
                      device_ms=res["device_ms"], epochs_total=int(res["passes"].sum()),
                      epochs_max_problem=int(res["passes"].sum(axis=1).max()),
                      epochs_max_lambda=int(res["passes"].max()),
                      converged=int(res["converged"].sum()), of=B * T)))
