"""Pin the CPU oracle (test infrastructure) to the reference.

* against the committed golden fixtures produced by the REAL reference
  (tests/golden/make_golden.py): bit for bit on this container's numpy/BLAS;
* against the reference's own inline known answers (pkg/tests/test_problem.py,
  test_regions.py, test_solver.py, test_path.py);
* directly against the reference package when /root/reference is importable.
"""

import os
import sys

import numpy as np
import pytest

from oracle import gapsafe_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
sys.path.insert(0, GOLD)
from make_golden import kernel_cases, path_cases  # noqa: E402


def test_kernels_match_reference_numba_bitwise():
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    k = kernel_cases()
    o = np.empty(k["cols"].size)
    O.tdot_dense(k["X"], k["v"], k["cols"], 0.0, o)
    assert np.array_equal(o, g["tdot_dense"])
    Xs = k["Xs"]
    o = np.empty(k["cols_s"].size)
    O.tdot_csc(Xs.data, Xs.indices, Xs.indptr, Xs.shape[0], k["v"], k["cols_s"], 0.0, o)
    assert np.array_equal(o, g["tdot_csc"])
    b, r = np.zeros(k["X"].shape[1]), k["v"].copy()
    for _ in range(7):
        O.cd_pass_dense(k["X"], b, r, k["cols"], k["lam"], k["nsq"], 0.0)
    assert np.array_equal(b, g["cd_dense_beta"]) and np.array_equal(r, g["cd_dense_rho"])
    b, r = np.zeros(k["X"].shape[1]), k["v"].copy()
    for _ in range(7):
        O.cd_pass_csc(Xs.data, Xs.indices, Xs.indptr, Xs.shape[0], b, r, k["cols_s"], k["lam_s"],
                      k["nsq_s"], 0.0)
    assert np.array_equal(b, g["cd_csc_beta"]) and np.array_equal(r, g["cd_csc_rho"])


@pytest.mark.parametrize("name", sorted(path_cases().keys()))
def test_oracle_path_matches_reference_golden(name):
    Xh, y, T, delta, eps = path_cases()[name]
    g = np.load(os.path.join(GOLD, name + ".npz"))
    X = O.DesignMatrix(Xh)
    lmax, _ = X.max_abs_correlation(y)
    grid = O.lambda_grid(lmax, T, delta)
    assert np.array_equal(grid, g["grid"])
    res = O.run_path(X, y, grid, O.SolverConfig(epsilon=eps, max_passes=100_000))
    assert np.array_equal(np.array([s.passes_done for s in res.states]), g["passes"])
    assert np.array_equal(res.betas, g["betas"])
    assert np.array_equal(np.array([c.gap for c in res.certs]), g["gaps"])
    traces = np.concatenate([np.array(t, dtype=np.float64).reshape(-1, 4) for t in res.traces])
    assert np.array_equal(traces, g["traces"])
    assert np.array_equal(np.concatenate([s.active for s in res.states]), g["actives"])
    assert np.array_equal(np.stack([s.theta.theta for s in res.states]), g["thetas"])


@pytest.mark.parametrize("name", ["rules_cfg0_p500", "rules_cfg3_n300_p2000"])
def test_oracle_rules_match_reference_golden(name):
    """static / dynamic / st3 / gap_dome (regions.py:159-273, solver.py:104-126):
    the oracle reproduces the reference's paths bit for bit."""
    from make_golden import RULES, rule_cases
    Xh, y, T, delta, eps = rule_cases()[name]
    g = np.load(os.path.join(GOLD, name + ".npz"))
    X = O.DesignMatrix(Xh)
    lmax, _ = X.max_abs_correlation(y)
    grid = O.lambda_grid(lmax, T, delta)
    assert np.array_equal(grid, g["grid"])
    for rule in RULES:
        res = O.run_path(X, y, grid, O.SolverConfig(epsilon=eps, max_passes=100_000, rule=rule))
        assert np.array_equal(np.array([s.passes_done for s in res.states]), g[f"{rule}__passes"]), rule
        assert np.array_equal(res.betas, g[f"{rule}__betas"]), rule
        assert np.array_equal(np.array([c.gap for c in res.certs]), g[f"{rule}__gaps"]), rule
        traces = np.concatenate([np.array(t, dtype=np.float64).reshape(-1, 4) for t in res.traces])
        assert np.array_equal(traces, g[f"{rule}__traces"]), rule
        assert np.array_equal(np.concatenate([s.active for s in res.states]), g[f"{rule}__actives"]), rule


def _diag(lam=1.0):
    return O.LassoProblem(O.DesignMatrix(np.array([[1.0, 0.0], [0.0, 2.0]])), np.array([1.0, 1.0]), lam)


def test_reference_known_answers():
    """Inline known answers of the reference tests, on the oracle."""
    prob = _diag()
    assert prob.lambda_max == 2.0 and prob.j_star == 1                 # test_problem.py:17-20
    assert O.primal_value(prob, np.zeros(2)) == 1.0                    # :32-33
    th = O.DualPoint(theta=np.array([0.5, 0.5]),
                     feasibility_margin=1.0 - prob.X.max_abs_correlation(np.array([0.5, 0.5]))[0])
    assert O.dual_value(prob, th) == pytest.approx(0.75)              # :63-66
    cert = O.duality_gap(prob, np.zeros(2), th)
    assert cert.gap == pytest.approx(0.25)                             # :82-88
    t = O.dual_scale(prob, prob.y)                                     # :105-109
    np.testing.assert_allclose(t.theta, [0.5, 0.5])
    assert t.feasibility_margin == pytest.approx(0.0, abs=1e-15)
    np.testing.assert_allclose(O.lambda_grid(2.0, 4, 3.0), [2.0, 0.2, 0.02, 0.002], rtol=1e-14)
    s = O.region_gap_sphere(prob, np.zeros(2), th)                     # test_regions.py:214-219
    assert s.radius == pytest.approx(np.sqrt(0.5))
    bad = O.DualPoint(theta=np.array([5.0, 5.0]), feasibility_margin=-9.0)
    with pytest.raises(O.InfeasibleDualError):
        O.dual_value(prob, bad)
    with pytest.raises(O.NumericalInconsistencyError):
        O.gap_radius(prob, -1.0)
    # single-feature closed form (test_solver.py:141-146)
    p1 = O.LassoProblem(O.DesignMatrix(np.array([[1.0], [1.0]])), np.array([2.0, 2.0]), 1.0)
    beta, cert, _ = O.solve(p1, O.SolverConfig(epsilon=1e-12))
    assert beta[0] == pytest.approx(1.5, abs=1e-9) and cert.gap <= 1e-12
    # lambda_max short-circuit (test_solver.py:133-139)
    p2 = _diag(lam=2.0)
    beta, cert, st = O.solve(p2, O.SolverConfig())
    assert np.all(beta == 0.0) and cert.gap == 0.0 and st.converged and st.passes_done == 0


def _reference():
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present (GPU box)")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import gapsafe
    return gapsafe


@pytest.mark.parametrize("seed,sparse", [(0, False), (1, True), (2, False)])
def test_oracle_equals_reference_directly(seed, sparse):
    G = _reference()
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    n, p = 30, 120
    Xh = rng.standard_normal((n, p))
    if sparse:
        Xh = sp.csc_matrix(Xh * (rng.random((n, p)) < 0.3))
    y = rng.standard_normal(n)
    D, Do = G.DesignMatrix(Xh), O.DesignMatrix(Xh)
    lmax, _ = D.max_abs_correlation(y)
    grid = G.lambda_grid(lmax, 8, 2.0)
    for rule in ("gap_sphere", "none"):
        a = G.run_path(D, y, grid, G.SolverConfig(epsilon=1e-10, rule=rule))
        b = O.run_path(Do, y, grid, O.SolverConfig(epsilon=1e-10, rule=rule))
        assert np.array_equal(a.betas, b.betas)
        assert [c.gap for c in a.certs] == [c.gap for c in b.certs]
        assert a.traces == b.traces


@pytest.mark.parametrize("k", [0, 1, 2])
def test_stacked_oracle_matches_reference_enet_golden(k):
    """F2: the oracle on the explicitly stacked design [X; sqrt(w) I] with the
    reference norms base_sq + w reproduces the reference's implicit-tail
    Elastic-Net solve (tests/golden/make_golden_enet.py): same passes, gap and
    beta (bit for bit dense; sparse within 1e-14, dense-vs-CSC base sums)."""
    from make_golden_enet import CASES, inputs
    g = np.load(os.path.join(GOLD, "enet_cfg0_p400.npz"))
    alpha, sparse = CASES[k]
    c, Xh = inputs(alpha, sparse)
    Xd = Xh.toarray() if sparse else Xh
    p = Xd.shape[1]
    lam = float(g[f"c{k}_lam"])
    tail = (1.0 - alpha) * lam
    Xo = O.DesignMatrix(np.vstack([Xd, np.sqrt(tail) * np.eye(p)]))
    Xo.col_norms_sq = np.einsum("ij,ij->j", Xd, Xd) + tail
    Xo.col_norms = np.sqrt(Xo.col_norms_sq)
    b, cert, st = O.solve(O.LassoProblem(Xo, np.concatenate([c.y, np.zeros(p)]), lam * alpha),
                          O.SolverConfig(epsilon=1e-10, max_passes=100_000))
    assert st.passes_done == int(g[f"c{k}_passes"])
    if sparse:
        np.testing.assert_allclose(b, g[f"c{k}_beta"], rtol=0, atol=1e-14)
    else:
        assert np.array_equal(b, g[f"c{k}_beta"]) and cert.gap == float(g[f"c{k}_gap"])
