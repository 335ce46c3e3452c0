"""Tiny workloads for compute-sanitizer (memcheck / racecheck / synccheck) on
the persistent kernels: k_solve (dense with a multi-warp CD chain, CSC) and
k_batch_path.   usage: python tools/sanitize_case.py dense|csc|batch"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth

what = sys.argv[1] if len(sys.argv) > 1 else "dense"
if what == "dense":
    rng = np.random.default_rng(5)
    n, p = 300, 500                              # R = 4, several CD warps
    X = synth.ar1_design(rng, n, p, 0.4)
    beta = np.zeros(p); beta[rng.choice(p, 10, replace=False)] = 1.0
    y = X @ beta + 0.2 * rng.standard_normal(n)
    D = gs.DesignMatrix(X)
    dev = gs.DeviceSolver(D, y)
    grid = gs.lambda_grid(dev.lambda_max, 4, 1.0)
    res = gs.run_path(D, y, grid, gs.SolverConfig(epsilon=1e-6 * float(y @ y), max_passes=2000), solver=dev)
    print("dense epochs", [s.passes_done for s in res.states])
elif what == "csc":
    c = synth.cfg3(n=400, p=2000, nnz_per_col=8)
    D = gs.DesignMatrix(c.X)
    dev = gs.DeviceSolver(D, c.y)
    grid = gs.lambda_grid(dev.lambda_max, 3, 0.7)
    res = gs.run_path(D, c.y, grid, gs.SolverConfig(epsilon=1e-5 * float(c.y @ c.y), max_passes=2000), solver=dev)
    print("csc epochs", [s.passes_done for s in res.states])
else:
    X0, y0, _ = synth.cfg4_shared(p=400)
    B = 3
    rows = np.stack([synth.cfg4_rows(b) for b in range(B)]).astype(np.int32)
    bs = gs.BatchPathSolver(gs.DesignMatrix(X0), y0, rows)
    grids = np.stack([gs.lambda_grid(bs.lambda_max[b], 3, 1.0) for b in range(B)])
    eps = np.array([1e-6 * float(y0[rows[b]] @ y0[rows[b]]) for b in range(B)])
    res = bs.run_paths(grids, gs.SolverConfig(epsilon=1.0, max_passes=2000), epsilons=eps)
    print("batch epochs", res["passes"].tolist())
