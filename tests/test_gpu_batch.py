"""Batched independent problems (BASELINE configs[4]): every problem's
device-side path equals the oracle's run_path on the same resampled rows."""

import numpy as np
import pytest

from oracle import gapsafe_oracle as O
from paper_1505_03410_b200 import synth
from parity import beta_close, gap_close

gs = pytest.importorskip("paper_1505_03410_b200")
pytestmark = pytest.mark.gpu


def test_batch_paths_match_oracle():
    rng = np.random.default_rng(11)
    X0 = synth.ar1_design(rng, 300, 1500, 0.5)
    beta = np.zeros(1500)
    beta[rng.choice(1500, 15, replace=False)] = rng.choice([-1.0, 1.0], 15)
    y0 = X0 @ beta + 0.3 * rng.standard_normal(300)
    B, n, T = 6, 150, 12
    rows = np.stack([np.random.default_rng([4, b]).integers(0, 300, n) for b in range(B)]).astype(np.int32)
    D0 = gs.DesignMatrix(X0)
    bs = gs.BatchPathSolver(D0, y0, rows)
    grids = np.stack([gs.lambda_grid(bs.lambda_max[b], T, 2.0) for b in range(B)])
    eps = np.array([1e-8 * float(y0[rows[b]] @ y0[rows[b]]) for b in range(B)])
    # configs[4]: every problem stops at its own tolerance eps_b = 1e-8 ||y_b||^2
    assert np.unique(eps).size == B
    res = bs.run_paths(grids, gs.SolverConfig(epsilon=1.0, max_passes=100_000), want_betas=True, epsilons=eps)
    for b in range(B):
        Xb = np.asfortranarray(X0[rows[b]])
        yb = y0[rows[b]]
        ref = O.run_path(O.DesignMatrix(Xb), yb, grids[b],
                         O.SolverConfig(epsilon=float(eps[b]), max_passes=100_000))
        yy = float(yb @ yb)
        for t in range(T):
            st = ref.states[t]
            assert res["passes"][b, t] == st.passes_done, (b, t)
            assert res["converged"][b, t] == st.converged
            assert res["n_active"][b, t] == st.active.size, (b, t)
            assert np.array_equal(np.flatnonzero(res["betas"][b, t]), np.flatnonzero(st.beta)), (b, t)
            assert beta_close(res["betas"][b, t], st.beta), (b, t)
            assert gap_close(res["gaps"][b, t], st.cert.gap, yy), (b, t)


def test_batch_more_problems_than_sms_schedule_independent():
    """The persistent batch grid (min(B, #SM) CTAs claiming problems from a
    counter) runs several problems per CTA when B > #SM; every problem's
    epochs, gaps and active sets equal those of a batch holding it alone."""
    X0, y0, _ = synth.cfg4_shared(p=1500)
    B = 160
    rows = np.stack([synth.cfg4_rows(b) for b in range(B)]).astype(np.int32)
    D0 = gs.DesignMatrix(X0)
    bs = gs.BatchPathSolver(D0, y0, rows)
    grids = np.stack([gs.lambda_grid(bs.lambda_max[b], 6, 1.5) for b in range(B)])
    cfg = gs.SolverConfig(epsilon=1e-8 * float(y0 @ y0) / 2, max_passes=100_000)
    res = bs.run_paths(grids, cfg)
    assert np.all(res["converged"])
    for b in (0, 77, 148, 159):
        one = gs.BatchPathSolver(D0, y0, rows[b:b + 1]).run_paths(grids[b:b + 1], cfg)
        assert np.array_equal(one["passes"][0], res["passes"][b]), b
        assert np.array_equal(one["gaps"][0], res["gaps"][b]), b
        assert np.array_equal(one["n_active"][0], res["n_active"][b]), b


def test_cfg4_full_width_per_problem_eps():
    """configs[4] at its stated width (the shared 1000 x 50000 design, n = 500
    bootstrap rows), B = 16 problems each at its own eps_b = 1e-8 ||y_b||^2,
    on the first grid points of the 50-lambda grid: two of the problems are
    checked against the oracle's run_path on the same resampled rows."""
    X0, y0, _ = synth.cfg4_shared()
    B, T, K = 16, 50, 14
    rows = np.stack([synth.cfg4_rows(b) for b in range(B)]).astype(np.int32)
    D0 = gs.DesignMatrix(X0)
    bs = gs.BatchPathSolver(D0, y0, rows)
    grids = np.stack([gs.lambda_grid(bs.lambda_max[b], T, 2.0)[:K] for b in range(B)])
    eps = np.array([1e-8 * float(y0[rows[b]] @ y0[rows[b]]) for b in range(B)])
    res = bs.run_paths(grids, gs.SolverConfig(epsilon=1.0, max_passes=100_000), want_betas=True, epsilons=eps)
    assert np.all(res["converged"])
    for b in (3, 12):
        Xb = np.asfortranarray(X0[rows[b]])
        yb = y0[rows[b]]
        ref = O.run_path(O.DesignMatrix(Xb), yb, grids[b], O.SolverConfig(epsilon=float(eps[b]), max_passes=100_000))
        yy = float(yb @ yb)
        for t in range(K):
            st = ref.states[t]
            assert res["passes"][b, t] == st.passes_done, (b, t)
            assert res["n_active"][b, t] == st.active.size, (b, t)
            assert np.array_equal(np.flatnonzero(res["betas"][b, t]), np.flatnonzero(st.beta)), (b, t)
            assert beta_close(res["betas"][b, t], st.beta), (b, t)
            assert gap_close(res["gaps"][b, t], st.cert.gap, yy), (b, t)
