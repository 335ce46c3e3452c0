"""Time one full Lasso path on the GPU (and optionally the oracle) for a config."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth

import argparse
ap = argparse.ArgumentParser()
ap.add_argument("name", nargs="?", default="cfg0")
ap.add_argument("p", nargs="?", type=int, default=None)
ap.add_argument("--once", action="store_true", help="time the first (cold) path only")
ap.add_argument("--lambdas", type=int, default=None, help="first T lambdas only")
ap.add_argument("--per-lambda", action="store_true", help="add per-lambda epochs / visits / uncertified / cd_ms")
a = ap.parse_args()
name = a.name
kw = {} if a.p is None else {"p": a.p}
c = synth.by_name(name, **kw)
t0 = time.perf_counter()
X = gs.DesignMatrix(c.X)
dev = gs.DeviceSolver(X, c.y)
grid = gs.lambda_grid(dev.lambda_max, c.n_lambdas, c.delta)[: a.lambdas]
cfg = gs.SolverConfig(epsilon=c.epsilon, max_passes=100_000)
t1 = time.perf_counter()
res = gs.run_path(X, c.y, grid, cfg, solver=dev)
t2 = time.perf_counter()
if not a.once:
    res = gs.run_path(X, c.y, grid, cfg, solver=dev)
t3 = time.perf_counter()
st = [s.stats for s in res.states]
out = dict(config=name, upload_s=t1 - t0, path_s_first=t2 - t1, path_s=(t3 - t2) if not a.once else (t2 - t1), lambdas=int(grid.size), n=int(c.X.shape[0]), p=int(c.X.shape[1]),
           epochs=int(sum(s.passes_done for s in res.states)),
           checkpoints=int(sum(x["checkpoints"] for x in st)),
           cd_visits=int(sum(x["cd_visits"] for x in st)),
           cd_uncertified=int(sum(x["cd_uncertified"] for x in st)),
           cd_nonzero=int(sum(x["cd_nonzero"] for x in st)),
           device_ms=float(sum(x["device_ms"] for x in st)),
           phase_ms={k: float(sum(x[k] for x in st)) for k in ("screen_ms", "ckpt_ms", "refresh_ms", "cd_ms")},
           refreshes=int(sum(x["n_refresh"] for x in st)),
           candidates=int(sum(x["cd_candidates"] for x in st)),
           skipped=int(sum(x["cd_skipped"] for x in st)),
           requeues=int(sum(x["cd_requeues"] for x in st)),
           converged=int(res.converged.sum()))
if a.per_lambda:
    out["per_lambda"] = [dict(t=t, epochs=int(s.passes_done), m_end=int(s.active.size), visits=int(x["cd_visits"]),
                              unc=int(x["cd_uncertified"]), nz=int(x["cd_nonzero"]), cd_ms=float(x["cd_ms"]),
                              refresh=int(x["n_refresh"]), refresh_ms=float(x["refresh_ms"]), ckpt_ms=float(x["ckpt_ms"]))
                         for t, (s, x) in enumerate(zip(res.states, st))]
print(json.dumps(out))
