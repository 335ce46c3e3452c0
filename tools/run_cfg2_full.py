"""BASELINE configs[2] at its stated size on ONE B200: 10,000 x 1,000,000 float32
(40 GB in HBM), 50 lambdas to lambda_max/20, gap tolerance 1e-5 ||y||^2.

The design is generated and uploaded block by block (synth.cfg2_streamed: the
host never holds more than one 400 MB block).  After the timed path:
  * the full-p screening pass is timed (algorithmic bytes / CUDA-event time);
  * parity at scale: for a few grid points the oracle re-runs
    the solve on the GPU path's own screened-in columns (downloaded from the
    device) with the path's lambda_max and the previous coefficients as warm
    start -- epochs, supports, coefficients and gaps must match -- and the
    sequential screen is re-checked by the oracle on a random column subsample
    with the GPU's own (theta, radius);
  * the final duality gap of every grid point is recomputed in float64 from
    the GPU's beta (X_S beta on the support columns, full X^T rho on the
    device) -- the "fp64 recheck of G".
    python tools/run_cfg2_full.py [p] [--check K]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("p", nargs="?", type=int, default=1_000_000)
ap.add_argument("--n", type=int, default=10_000)
ap.add_argument("--block", type=int, default=10_000)
ap.add_argument("--check", type=int, default=3, help="grid points re-solved by the oracle")
ap.add_argument("--sub", type=int, default=20_000, help="random columns for the screen re-check")
a = ap.parse_args()
n, p = a.n, a.p

t0 = time.perf_counter()
holder = {}
# stream: upload each block as it is generated (one block resident on the host)
class Stream:
    def __iter__(self):
        import threading, queue
        q = queue.Queue(maxsize=1)
        def work():
            holder["res"] = synth.cfg2_streamed(p=p, n=n, block=a.block, on_block=lambda b0, Xb: q.put((b0, Xb)))
            q.put(None)
        th = threading.Thread(target=work, daemon=True)
        th.start()
        while True:
            item = q.get()
            if item is None:
                break
            yield item
        th.join()
X = gs.DesignMatrix.from_blocks(n, p, np.float32, Stream())
_, y, beta_star, meta = holder["res"]
t1 = time.perf_counter()
dev = gs.DeviceSolver(X, y)
grid = gs.lambda_grid(dev.lambda_max, 50, float(np.log10(20.0)))
eps = 1e-5 * float(y @ y)
cfg = gs.SolverConfig(epsilon=eps, max_passes=100_000)
t2 = time.perf_counter()
res = gs.run_path(X, y, grid, cfg, solver=dev)
t3 = time.perf_counter()
st = [s.stats for s in res.states]
out = dict(config="cfg2", n=n, p=p, hbm_bytes=int(X.device_bytes), gen_upload_s=t1 - t0, setup_s=t2 - t1, path_s=t3 - t2,
           lambdas=int(grid.size), epochs=int(sum(s.passes_done for s in res.states)), converged=int(res.converged.sum()),
           active_end=[int(s.active.size) for s in res.states][::7],
           phase_ms={k: float(sum(x[k] for x in st)) for k in ("screen_ms", "ckpt_ms", "refresh_ms", "cd_ms")},
           n_screen=int(sum(x["n_screen"] for x in st)), cd_uncertified=int(sum(x["cd_uncertified"] for x in st)),
           cd_visits=int(sum(x["cd_visits"] for x in st)))
# ---- the screening pass, timed alone
byts = n * p * 4 + 9 * p + 8 * n
ms = gs.PathTimer.screen_pass_ms(X, res.states[-1].theta.theta, 1e-3, reps=10)
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    peak = 6650.0
out["screen"] = dict(ms=ms, bytes=byts, gbs=byts / ms / 1e6, frac=byts / ms / 1e6 / peak, peak=peak,
                     in_path_ms=out["phase_ms"]["screen_ms"] / max(1, out["n_screen"]))
print(json.dumps(out), flush=True)

# ---- parity at scale
from oracle import gapsafe_oracle as O
par = []
T = grid.size
for t in sorted(set(np.linspace(1, T - 1, a.check).astype(int).tolist())):
    stt, prev = res.states[t], res.states[t - 1]
    # (1) the sequential screen on a random column subsample, oracle arithmetic, the GPU's own inputs
    rng = np.random.default_rng([22, t])
    sub = np.sort(rng.choice(p, size=min(a.sub, p), replace=False))
    Xs = X.columns_to_host(sub).astype(np.float64)
    lam = float(grid[t])
    rho_p, th_p, beta_p = prev.residual, prev.theta.theta, prev.beta
    primal = 0.5 * float(rho_p @ rho_p) + lam * float(np.abs(beta_p).sum())
    diff = th_p - y / lam
    dual = 0.5 * float(y @ y) - 0.5 * lam ** 2 * float(diff @ diff)
    r = float(np.sqrt(2.0 * max(primal - dual, 0.0)) / lam)
    scr = O.screen(O.Sphere(center=th_p, radius=r), O.DesignMatrix(Xs))
    kept_oracle = sub[scr.active_set]
    # the GPU's own survivors of this screen: the same fused pass on the same inputs
    A0 = gs.PathTimer.screen_pass_active(X, th_p, r)
    near = np.abs(scr.mu - (1 - 1e-9)) <= 1e-10
    diff_cols = np.setxor1d(np.intersect1d(A0, sub), kept_oracle)
    screen_equal = bool(np.all(near[np.searchsorted(sub, diff_cols)])) if diff_cols.size else True
    # (2) the oracle's solve on exactly those columns, the path's lambda_max, warm start = previous beta
    XA = X.columns_to_host(A0).astype(np.float64)
    prob = O.LassoProblem(O.DesignMatrix(XA), y, lam, lambda_max=(dev.lambda_max, 0))
    bA, cert, so = O.solve(prob, O.SolverConfig(epsilon=eps, max_passes=100_000), warm_beta=beta_p[A0],
                           active0=np.arange(A0.size, dtype=np.int64))
    bfull = np.zeros(p); bfull[A0] = bA
    scale = max(1.0, float(np.max(np.abs(stt.beta))))
    par.append(dict(t=int(t), lam=lam, screen_subsample=int(sub.size), screen_kept_oracle=int(kept_oracle.size),
                    screen_masks_equal_on_subsample=screen_equal, near_threshold=int(near.sum()),
                    screened_in=int(A0.size), epochs_gpu=int(stt.passes_done), epochs_oracle=int(so.passes_done),
                    epochs_equal=bool(stt.passes_done == so.passes_done),
                    active_equal=bool(np.array_equal(A0[so.active], stt.active)),
                    support_equal=bool(np.array_equal(np.flatnonzero(bfull), np.flatnonzero(stt.beta))),
                    beta_rel_diff=float(np.max(np.abs(bfull - stt.beta)) / scale),
                    gap_gpu=float(stt.cert.gap), gap_oracle=float(cert.gap), eps=eps))
    print(json.dumps(par[-1]), flush=True)
# ---- fp64 recheck of the final gap of every grid point from the GPU's beta
rechk = []
for t in range(T):
    stt = res.states[t]
    lam = float(grid[t])
    S = np.flatnonzero(stt.beta)
    XS = X.columns_to_host(S).astype(np.float64) if S.size else np.zeros((n, 0))
    rho = y - XS @ stt.beta[S]
    corr, _ = X.max_abs_correlation(rho)          # full-p |X^T rho|_inf on the device (f64 arithmetic)
    alpha = float(y @ rho) / (lam * float(rho @ rho)) if float(rho @ rho) > 0 else 0.0
    if corr > 0:
        alpha = min(max(alpha, -1.0 / corr), 1.0 / corr)
    theta = alpha * rho
    diff = theta - y / lam
    G = 0.5 * float(rho @ rho) + lam * float(np.abs(stt.beta).sum()) - (0.5 * float(y @ y) - 0.5 * lam ** 2 * float(diff @ diff))
    rechk.append(dict(t=t, gap_full_dual=G, gap_reported=float(stt.cert.gap), le_eps=bool(G <= eps * (1 + 1e-6) + 64 * 2.2e-16 * float(y @ y))))
print(json.dumps(dict(parity=par, gap_recheck_all_le_eps=bool(all(r["le_eps"] for r in rechk)),
                      gap_recheck_max_ratio=float(max(r["gap_full_dual"] for r in rechk) / eps), gap_recheck=rechk[::7])))
