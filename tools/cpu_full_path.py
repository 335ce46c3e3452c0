"""Time the CPU oracle (bit-identical restatement of the reference) on a full
config path; writes a JSON record.  Test/measurement infrastructure only."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import gapsafe_oracle as O
from paper_1505_03410_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
c = synth.by_name(name)
X = O.DesignMatrix(c.X)
lmax, _ = X.max_abs_correlation(c.y)
grid = O.lambda_grid(lmax, c.n_lambdas, c.delta)
t0 = time.perf_counter()
res = O.run_path(X, c.y, grid, O.SolverConfig(epsilon=c.epsilon, max_passes=100_000))
wall = time.perf_counter() - t0
print(json.dumps(dict(config=name, wall_s=wall, run_path_timings_s=sum(res.timings),
                      epochs=int(sum(s.passes_done for s in res.states)),
                      per_lambda_s=[round(x, 4) for x in res.timings],
                      converged=int(res.converged.sum()), cores=len(os.sched_getaffinity(0)),
                      host="build container (Intel Xeon, 8 cores, OpenBLAS 8 threads)")))
