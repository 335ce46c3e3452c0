"""Short path for profiling: first T lambdas of a config (default cfg0, 30)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "cfg0"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kw = {"p": int(sys.argv[3])} if len(sys.argv) > 3 else {}
c = synth.by_name(name, **kw)
X = gs.DesignMatrix(c.X)
dev = gs.DeviceSolver(X, c.y)
grid = gs.lambda_grid(dev.lambda_max, c.n_lambdas, c.delta)[:T]
res = gs.run_path(X, c.y, grid, gs.SolverConfig(epsilon=c.epsilon, max_passes=100_000), solver=dev)
print("epochs", sum(s.passes_done for s in res.states), "converged", int(res.converged.sum()))
