"""Generate golden fixtures by running the REAL reference implementation.

Run in the build container, where /root/reference is importable:

    python tests/golden/make_golden.py

It imports ``gapsafe`` from /root/reference/pkg/src (read-only; numba caches
in a user dir) and writes small .npz files next to this script.  The GPU box
has no /root/reference, so the tests read only these committed fixtures.

Fixtures:
  kernels.npz   -- _kernels.tdot_dense / tdot_csc / cd_pass_dense / cd_pass_csc
                   on seeded inputs (the numba kernels themselves);
  path_*.npz    -- full run_path results (betas, per-lambda epochs, traces,
                   certificates, final active sets) on seeded cases built by
                   paper_1505_03410_b200.synth at reduced sizes.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"


def _import_reference():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gapsafe                      # noqa: F401
    from gapsafe import _kernels        # noqa: F401
    return gapsafe


def kernel_cases():
    """Seeded inputs shared by make_golden and the tests."""
    rng = np.random.default_rng(1234)
    n, p = 57, 211
    X = np.asfortranarray(rng.standard_normal((n, p)))
    v = rng.standard_normal(n)
    cols = np.sort(rng.choice(p, 150, replace=False)).astype(np.int64)
    nsq = np.einsum("ij,ij->j", X, X)
    lam = 0.2 * float(np.max(np.abs(X.T @ v)))
    Xs = sp.random(n, p, density=0.15, random_state=np.random.RandomState(7), format="csc")
    Xs.sort_indices()
    nsq_s = np.asarray(Xs.multiply(Xs).sum(axis=0)).ravel()
    cols_s = np.flatnonzero(nsq_s > 0).astype(np.int64)
    lam_s = 0.2 * float(np.max(np.abs(Xs.T @ v)))
    return dict(X=X, v=v, cols=cols, nsq=nsq, lam=lam, Xs=Xs, nsq_s=nsq_s, cols_s=cols_s, lam_s=lam_s)


def path_cases():
    sys.path.insert(0, ROOT)
    from paper_1505_03410_b200 import synth
    c0 = synth.cfg0(p=600)
    c1 = synth.cfg1(p=1500, n=200)
    c3 = synth.cfg3(p=3000, n=400, nnz_per_col=12)
    return {
        "path_cfg0_p600": (c0.X, c0.y, 12, 3.0, c0.epsilon),
        "path_cfg1_n200_p1500": (c1.X, c1.y, 10, 2.0, c1.epsilon),
        "path_cfg3_n400_p3000": (c3.X, c3.y, 10, 2.0, c3.epsilon),
    }


RULES = ("static", "dynamic", "st3", "gap_dome")


def rule_cases():
    """Every non-default screening rule on a dense and a CSC case."""
    sys.path.insert(0, ROOT)
    from paper_1505_03410_b200 import synth
    c0 = synth.cfg0(p=500)
    c3 = synth.cfg3(p=2000, n=300, nnz_per_col=10)
    return {
        "rules_cfg0_p500": (c0.X, c0.y, 8, 2.0, c0.epsilon),
        "rules_cfg3_n300_p2000": (c3.X, c3.y, 8, 2.0, c3.epsilon),
    }


def _record(res, eps):
    traces = [np.array(t, dtype=np.float64).reshape(-1, 4) for t in res.traces]
    return dict(betas=res.betas, epsilon=np.float64(eps),
                passes=np.array([s.passes_done for s in res.states]),
                gaps=np.array([c.gap for c in res.certs]),
                converged=res.converged,
                trace_rows=np.array([t.shape[0] for t in traces]),
                traces=np.concatenate(traces),
                active_sizes=np.array([s.active.size for s in res.states]),
                actives=np.concatenate([s.active for s in res.states]))


def main_rules():
    G = _import_reference()
    for name, (Xh, y, T, delta, eps) in rule_cases().items():
        D = G.DesignMatrix(Xh)
        lmax, _ = D.max_abs_correlation(y)
        grid = G.lambda_grid(lmax, T, delta)
        rec = {"grid": grid}
        for rule in RULES:
            res = G.run_path(D, y, grid, G.SolverConfig(epsilon=eps, max_passes=100_000, rule=G.Rule(rule)))
            for k2, v2 in _record(res, eps).items():
                rec[f"{rule}__{k2}"] = v2
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
        print(name, {r: int(rec[f"{r}__passes"].sum()) for r in RULES})


def main():
    G = _import_reference()
    from gapsafe import _kernels as K
    k = kernel_cases()
    out = {}
    o = np.empty(k["cols"].size)
    K.tdot_dense(k["X"], k["v"], k["cols"], 0.0, o)
    out["tdot_dense"] = o.copy()
    Xs = k["Xs"]
    o = np.empty(k["cols_s"].size)
    K.tdot_csc(Xs.data, Xs.indices, Xs.indptr, Xs.shape[0], k["v"], k["cols_s"], 0.0, o)
    out["tdot_csc"] = o.copy()
    b, r = np.zeros(k["X"].shape[1]), k["v"].copy()
    for _ in range(7):
        K.cd_pass_dense(k["X"], b, r, k["cols"], k["lam"], k["nsq"], 0.0)
    out["cd_dense_beta"], out["cd_dense_rho"] = b.copy(), r.copy()
    b, r = np.zeros(k["X"].shape[1]), k["v"].copy()
    for _ in range(7):
        K.cd_pass_csc(Xs.data, Xs.indices, Xs.indptr, Xs.shape[0], b, r, k["cols_s"], k["lam_s"],
                      k["nsq_s"], 0.0)
    out["cd_csc_beta"], out["cd_csc_rho"] = b.copy(), r.copy()
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("kernels.npz", {a: v.shape for a, v in out.items()})

    for name, (Xh, y, T, delta, eps) in path_cases().items():
        D = G.DesignMatrix(Xh)
        lmax, _ = D.max_abs_correlation(y)
        grid = G.lambda_grid(lmax, T, delta)
        res = G.run_path(D, y, grid, G.SolverConfig(epsilon=eps, max_passes=100_000))
        traces = [np.array(t, dtype=np.float64).reshape(-1, 4) for t in res.traces]
        rec = dict(grid=grid, betas=res.betas, epsilon=np.float64(eps),
                   passes=np.array([s.passes_done for s in res.states]),
                   gaps=np.array([c.gap for c in res.certs]),
                   primals=np.array([c.primal for c in res.certs]),
                   converged=res.converged,
                   trace_rows=np.array([t.shape[0] for t in traces]),
                   traces=np.concatenate(traces),
                   active_sizes=np.array([s.active.size for s in res.states]),
                   actives=np.concatenate([s.active for s in res.states]),
                   thetas=np.stack([s.theta.theta for s in res.states]))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
        print(name, "epochs", int(rec["passes"].sum()), "converged", bool(np.all(res.converged)))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "rules":
        main_rules()
    else:
        main()
        main_rules()
