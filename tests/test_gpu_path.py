"""Path-level parity: solve / run_path on the B200 against the CPU oracle
(a bit-identical restatement of the reference, tests/test_oracle_golden.py),
on the same seeded inputs.  See tests/parity.py for the criteria."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gapsafe_oracle as O
from paper_1505_03410_b200 import synth
from parity import compare_paths, compare_states

gs = pytest.importorskip("paper_1505_03410_b200")
pytestmark = pytest.mark.gpu


def _paths(Xh, y, T, delta, eps, rule="gap_sphere", max_passes=100_000, f=10, certify=True):
    X = gs.DesignMatrix(Xh)
    dev = gs.DeviceSolver(X, y)
    Xo = O.DesignMatrix(Xh)
    lmax, _ = Xo.max_abs_correlation(y)
    grid = O.lambda_grid(lmax, T, delta)
    ra = gs.run_path(X, y, grid, gs.SolverConfig(epsilon=eps, max_passes=max_passes, screen_every=f,
                                                 rule=rule, certify=certify), solver=dev)
    rb = O.run_path(Xo, y, grid, O.SolverConfig(epsilon=eps, max_passes=max_passes, screen_every=f,
                                                rule=rule))
    return ra, rb, float(y @ y)


@pytest.mark.parametrize("rule", ["gap_sphere", "none"])
def test_path_cfg0_shape_small_p(rule):
    c = synth.cfg0(p=1500)
    ra, rb, yy = _paths(c.X, c.y, 20, 3.0, c.epsilon, rule=rule)
    compare_paths(ra, rb, yy)


def test_path_cfg0_full():
    """configs[0] at full size (72 x 7129, 100 lambdas to lambda_max/1e3)."""
    c = synth.cfg0()
    ra, rb, yy = _paths(c.X, c.y, c.n_lambdas, c.delta, c.epsilon)
    compare_paths(ra, rb, yy)
    assert np.all(ra.converged)


@pytest.mark.parametrize("gram", ["0", "1", "2"])
def test_path_no_certify_identical_to_certify(gram, monkeypatch):
    """Certified-zero skipping is exact.  With one reduction per coordinate
    (GS_CD_GRAM=0) the paths with and without it are bit-identical.  The
    Gram-window consumer groups the coordinates it computes into windows, so
    skipping changes the window partition and hence roundings (never an
    update): epochs, traces' active-set sizes and supports are identical and
    the coefficients agree to round-off."""
    monkeypatch.setenv("GS_CD_GRAM", gram)
    c = synth.cfg0(p=800)
    X = gs.DesignMatrix(c.X)
    dev = gs.DeviceSolver(X, c.y)
    grid = gs.lambda_grid(dev.lambda_max, 15, 2.5)
    a = gs.run_path(X, c.y, grid, gs.SolverConfig(epsilon=c.epsilon, max_passes=100_000), solver=dev)
    b = gs.run_path(X, c.y, grid, gs.SolverConfig(epsilon=c.epsilon, max_passes=100_000, certify=False),
                    solver=dev)
    if gram == "0":
        assert np.array_equal(a.betas, b.betas)
        assert [x.gap for x in a.certs] == [x.gap for x in b.certs]
        assert a.traces == b.traces
    else:
        assert [s.passes_done for s in a.states] == [s.passes_done for s in b.states]
        assert [[r[:2] for r in t] for t in a.traces] == [[r[:2] for r in t] for t in b.traces]
        assert np.array_equal(a.betas != 0, b.betas != 0)
        np.testing.assert_allclose(a.betas, b.betas, rtol=0, atol=1e-12 * np.abs(b.betas).max())


@pytest.mark.parametrize("gram", ["0", "1", "2"])
def test_path_cd_modes_match_oracle(gram, monkeypatch):
    """Both CD consumers (Gram windows, one reduction per coordinate) meet the
    parity criteria against the oracle on the cfg0 generator."""
    monkeypatch.setenv("GS_CD_GRAM", gram)
    c = synth.cfg0(p=2000)
    ra, rb, yy = _paths(c.X, c.y, 25, 3.0, c.epsilon)
    compare_paths(ra, rb, yy)


def test_path_deterministic_bit_identical():
    """pkg/tests/test_path.py:124-131 on the device."""
    c = synth.cfg0(p=900)
    X = gs.DesignMatrix(c.X)
    grid = gs.lambda_grid(gs.DeviceSolver(X, c.y).lambda_max, 10, 3.0)
    cfg = gs.SolverConfig(epsilon=1e-8, max_passes=100_000)
    a = gs.run_path(X, c.y, grid, cfg)
    b = gs.run_path(X, c.y, grid, cfg)
    assert np.array_equal(a.betas, b.betas)
    assert [x.gap for x in a.certs] == [x.gap for x in b.certs]


def test_path_cfg1_shape_reduced():
    """configs[1] generator at reduced width (1000 x 4000)."""
    c = synth.cfg1(p=4000)
    ra, rb, yy = _paths(c.X, c.y, 12, 2.0, c.epsilon)
    compare_paths(ra, rb, yy)


def test_path_float32_storage():
    """fp32 storage / fp64 arithmetic == the oracle on the upcast values."""
    c = synth.cfg0(p=700)
    X32 = np.asfortranarray(c.X.astype(np.float32))
    X64 = np.asfortranarray(X32.astype(np.float64))
    X = gs.DesignMatrix(X32)
    Xo = O.DesignMatrix(X64)
    lmax, _ = Xo.max_abs_correlation(c.y)
    grid = O.lambda_grid(lmax, 10, 2.0)
    ra = gs.run_path(X, c.y, grid, gs.SolverConfig(epsilon=c.epsilon, max_passes=100_000))
    rb = O.run_path(Xo, c.y, grid, O.SolverConfig(epsilon=c.epsilon, max_passes=100_000))
    compare_paths(ra, rb, float(c.y @ c.y))


def test_path_sparse_csc():
    c = synth.cfg3(p=20_000, n=2_000, nnz_per_col=20)
    ra, rb, yy = _paths(c.X, c.y, 15, 2.0, c.epsilon)
    compare_paths(ra, rb, yy)


def test_solve_single_lambda_and_hooks():
    c = synth.cfg0(p=500)
    X = gs.DesignMatrix(c.X)
    prob = gs.LassoProblem(X, c.y, 0.1 * gs.DeviceSolver(X, c.y).lambda_max)
    seen = []
    cfg = gs.SolverConfig(epsilon=1e-10, max_passes=100_000, track_active=True,
                          on_checkpoint=lambda a: seen.append(a.size))
    beta, cert, st = gs.solve(prob, cfg)
    Xo = O.DesignMatrix(c.X)
    po = O.LassoProblem(Xo, c.y, prob.lam)
    b2, c2, st2 = O.solve(po, O.SolverConfig(epsilon=1e-10, max_passes=100_000, track_active=True))
    compare_states(st, st2, float(c.y @ c.y))
    assert len(st.active_history) == len(st2.active_history)
    for a, b in zip(st.active_history, st2.active_history):
        assert np.array_equal(a, b)
    assert seen == [a.size for a in st2.active_history]


def test_solve_budget_exhausted():
    c = synth.cfg0(p=300)
    X = gs.DesignMatrix(c.X)
    lam = 0.01 * gs.DeviceSolver(X, c.y).lambda_max
    prob = gs.LassoProblem(X, c.y, lam)
    beta, cert, st = gs.solve(prob, gs.SolverConfig(epsilon=1e-14, max_passes=3))
    po = O.LassoProblem(O.DesignMatrix(c.X), c.y, lam)
    _, _, st2 = O.solve(po, O.SolverConfig(epsilon=1e-14, max_passes=3))
    assert not st.converged and not st2.converged
    compare_states(st, st2, float(c.y @ c.y))


def test_solve_warm_start_and_active0():
    c = synth.cfg0(p=400)
    X = gs.DesignMatrix(c.X)
    lam = 0.2 * gs.DeviceSolver(X, c.y).lambda_max
    prob = gs.LassoProblem(X, c.y, lam)
    b0, _, _ = gs.solve(prob, gs.SolverConfig(epsilon=1e-12, max_passes=100_000))
    _, _, st = gs.solve(prob, gs.SolverConfig(epsilon=1e-8), warm_beta=b0)
    assert st.converged and st.passes_done == 0
    warm = np.ones(400)
    keep = np.array([0, 3, 7])
    beta, _, _ = gs.solve(prob, gs.SolverConfig(epsilon=1e-300, max_passes=1), warm_beta=warm,
                          active0=keep)
    assert np.all(beta[np.setdiff1d(np.arange(400), keep)] == 0.0)


def test_lambda_max_shortcut():
    c = synth.cfg0(p=300)
    X = gs.DesignMatrix(c.X)
    dev = gs.DeviceSolver(X, c.y)
    prob = gs.LassoProblem(X, c.y, dev.lambda_max)
    beta, cert, st = gs.solve(prob, gs.SolverConfig())
    assert np.all(beta == 0) and cert.gap == 0.0 and st.converged and st.passes_done == 0
    po = O.LassoProblem(O.DesignMatrix(c.X), c.y, prob.lam)
    _, _, st2 = O.solve(po, O.SolverConfig())
    assert np.array_equal(st.active, st2.active)
    assert st.screen_trace == [(0, st2.active.size, 0.0, 0.0)]


def test_errors_map_to_reference_exceptions():
    X = gs.DesignMatrix(np.array([[1.0, 0.0], [0.0, 2.0]]))
    prob = gs.LassoProblem(X, np.array([1.0, 1.0]), 1.0)
    th = gs.make_dual_point(X, np.array([5.0, 5.0]))
    with pytest.raises(gs.InfeasibleDualError):
        gs.dual_value(prob, th)
    with pytest.raises(ValueError):
        gs.LassoProblem(X, np.array([1.0, 1.0]), 2.5)
    with pytest.raises(gs.NumericalInconsistencyError):
        gs.gap_radius(prob, -1.0)
    with pytest.raises(gs.NumericalInconsistencyError):
        gs.region_gap_dome(prob, np.array([0.0, 0.0]), gs.make_dual_point(X, np.array([0.5, 0.5])),
                           residual=np.array([0.0, 0.0]))
    with pytest.raises(ValueError):
        gs.region_dynamic(prob, th)


def test_problem_algebra_hand_values():
    """pkg/tests/test_problem.py known answers on the 2x2 diagonal problem."""
    X = gs.DesignMatrix(np.array([[1.0, 0.0], [0.0, 2.0]]))
    prob = gs.LassoProblem(X, np.array([1.0, 1.0]), 1.0)
    assert prob.lambda_max == 2.0 and prob.j_star == 1
    assert gs.primal_value(prob, np.zeros(2)) == 1.0
    th = gs.make_dual_point(X, np.array([0.5, 0.5]))
    assert gs.dual_value(prob, th) == pytest.approx(0.75)
    cert = gs.duality_gap(prob, np.zeros(2), th)
    assert cert.gap == pytest.approx(0.25)
    s = gs.region_gap_sphere(prob, np.zeros(2), th)
    assert s.radius == pytest.approx(np.sqrt(0.5))
    t = gs.dual_scale(prob, prob.y)
    np.testing.assert_allclose(t.theta, [0.5, 0.5])
    assert t.feasibility_margin == pytest.approx(0.0, abs=1e-15)
    assert gs.dual_scale(prob, np.zeros(2)).interpolating


def _ragged_csc(seed, n, p, max_nnz):
    """CSC with column lengths 1..max_nnz (some above 32: such columns run
    alone in their wave), lognormal values, unit norms."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, max_nnz + 1, size=p)
    rows = [np.sort(rng.choice(n, size=k, replace=False)) for k in lens]
    vals = [rng.lognormal(size=k) for k in lens]
    vals = [v / np.linalg.norm(v) for v in vals]
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    X = sp.csc_matrix((np.concatenate(vals), np.concatenate(rows).astype(np.int32), indptr), shape=(n, p))
    beta = np.zeros(p)
    beta[rng.choice(p, 40, replace=False)] = rng.choice([-1.0, 1.0], 40)
    y = X @ beta
    y += rng.standard_normal(n) * np.linalg.norm(y) / np.sqrt(n) / 4
    return X, y


@pytest.mark.parametrize("n,p,max_nnz", [(400, 3000, 12), (1500, 6000, 60), (5000, 8000, 30)])
def test_path_sparse_waves_ragged(n, p, max_nnz):
    """Conflict-free wave CD on ragged CSC columns (row conflicts, long
    columns, rollbacks) against the oracle path."""
    X, y = _ragged_csc(n + p, n, p, max_nnz)
    ra, rb, yy = _paths(X, y, 12, 2.0, 1e-8 * float(y @ y))
    compare_paths(ra, rb, yy)


def test_path_sparse_certify_identical():
    """Certified skipping and rollback are exact on the CSC path too."""
    X, y = _ragged_csc(7, 1200, 5000, 40)
    Xd = gs.DesignMatrix(X)
    dev = gs.DeviceSolver(Xd, y)
    grid = gs.lambda_grid(dev.lambda_max, 12, 2.0)
    eps = 1e-8 * float(y @ y)
    a = gs.run_path(Xd, y, grid, gs.SolverConfig(epsilon=eps, max_passes=100_000), solver=dev)
    b = gs.run_path(Xd, y, grid, gs.SolverConfig(epsilon=eps, max_passes=100_000, certify=False), solver=dev)
    assert np.array_equal(a.betas, b.betas)
    assert [x.gap for x in a.certs] == [x.gap for x in b.certs]


@pytest.mark.parametrize("n, p, T", [(2000, 1500, 10), (10_000, 3000, 12)])
def test_path_cfg2_generator_long_columns(n, p, T):
    """configs[2] generator (float32 storage, unit-norm N(0,1) columns, tol 1e-5,
    grid to lambda_max / 20) at long column lengths: the 48-rows-per-lane CD
    with columns streamed from the shared-memory ring, against the oracle on
    the upcast values."""
    c = synth.cfg2(p=p, n=n, k=min(500, p // 4))
    X64 = np.asfortranarray(c.X.astype(np.float64))
    X = gs.DesignMatrix(c.X)
    Xo = O.DesignMatrix(X64)
    lmax, _ = Xo.max_abs_correlation(c.y)
    grid = O.lambda_grid(lmax, T, c.delta)
    ra = gs.run_path(X, c.y, grid, gs.SolverConfig(epsilon=c.epsilon, max_passes=100_000))
    rb = O.run_path(Xo, c.y, grid, O.SolverConfig(epsilon=c.epsilon, max_passes=100_000))
    compare_paths(ra, rb, float(c.y @ c.y))
    assert np.all(ra.converged)


@pytest.mark.parametrize("rule", ["static", "dynamic", "st3", "gap_dome"])
@pytest.mark.parametrize("kind", ["dense", "csc"])
def test_path_rules_match_oracle(rule, kind):
    """Every screening rule of the reference on the
    device: same epochs, traces (incl. each rule's trace radius), active sets
    and supports as the oracle, coefficients and gaps within tolerance."""
    if kind == "dense":
        c = synth.cfg0(p=1200)
    else:
        c = synth.cfg3(p=3000, n=400, nnz_per_col=12)
    ra, rb, yy = _paths(c.X, c.y, 12, 2.5, c.epsilon, rule=rule)
    compare_paths(ra, rb, yy)
    if rule != "gap_dome":
        # static / dynamic / ST3 traces report the region radius (solver.py:122-126);
        # the dome's is the gap radius, covered by the gap criterion
        for ta, tb in zip(ra.traces, rb.traces):
            for x, y in zip(ta, tb):
                assert abs(x[3] - y[3]) <= 1e-9 * max(1.0, abs(y[3])), (rule, x, y)


def test_regions_api_dome_and_spheres_match_oracle():
    """Region constructors and the dome test through the public API
    (regions.py:82-119, 159-273) against the oracle."""
    c = synth.cfg0(p=900)
    X = gs.DesignMatrix(c.X)
    Xo = O.DesignMatrix(c.X)
    lmax, _ = Xo.max_abs_correlation(c.y)
    lam = 0.3 * lmax
    cfg = gs.SolverConfig(epsilon=c.epsilon, max_passes=40, screen_every=10)
    prob = gs.LassoProblem(X, c.y, lam)
    beta, cert, st = gs.solve(prob, cfg)
    po = O.LassoProblem(Xo, c.y, lam)
    th = O.DualPoint(theta=st.theta.theta, feasibility_margin=st.theta.feasibility_margin)
    for mk, mko in ((lambda: gs.region_static(prob), lambda: O.region_static(po)),
                    (lambda: gs.region_dynamic(prob, st.theta), lambda: O.region_dynamic(po, th)),
                    (lambda: gs.region_st3(prob, st.theta), lambda: O.region_st3(po, th)),
                    (lambda: gs.region_gap_dome(prob, beta, st.theta, residual=st.residual),
                     lambda: O.region_gap_dome(po, beta, th, residual=st.residual))):
        a, b = mk(), mko()
        mu_a, mu_b = gs.mu_values(a, X), O.mu_values(b, Xo)
        np.testing.assert_allclose(mu_a, mu_b, rtol=1e-10, atol=1e-12)
        sa, sb = gs.screen(a, X), O.screen(b, Xo)
        near = np.abs(mu_b - (1 - gs.SCREEN_SAFETY)) <= 1e-10
        assert np.all(near[np.setxor1d(sa.active_set, sb.active_set)])


def test_elastic_net_pure_l1_and_kkt():
    """elastic_net.py: the pure-l1 reduction is the plain Lasso, and a converged
    path point satisfies the KKT conditions to the gap tolerance."""
    c = synth.cfg0(p=700)
    X = gs.DesignMatrix(c.X)
    lmax, _ = X.max_abs_correlation(c.y)
    en = gs.ElasticNetProblem(X, c.y, 0.2 * lmax, 1.0)
    prob = gs.to_lasso(en)
    assert prob.lam == 0.2 * lmax and prob.X is X
    beta, cert, st = gs.solve(prob, gs.SolverConfig(epsilon=1e-12 * float(c.y @ c.y), max_passes=100_000))
    assert st.converged
    assert gs.kkt_residual(en, beta) <= 1e-5 * prob.lam
    ob = gs.objective(en, beta)
    assert abs(ob - cert.primal) <= 1e-9 * abs(ob)


def test_tail_behaves_like_stacked_identity():
    """design_matrix.py:54-65,100-183 with tail_weight > 0 (test_design_matrix.py:135-150)."""
    rng = np.random.default_rng(4)
    base = rng.standard_normal((6, 4))
    w = 0.7
    for storage in (base, sp.csc_matrix(base)):
        X = gs.DesignMatrix(storage, tail_weight=w)
        explicit = np.vstack([base, np.sqrt(w) * np.eye(4)])
        assert X.n_rows == 10 and X.tail_scale == float(np.sqrt(w))
        np.testing.assert_allclose(X.toarray(), explicit, rtol=1e-15)
        v = rng.standard_normal(10)
        for j in range(4):
            assert X.col_dot(j, v) == pytest.approx(explicit[:, j] @ v, rel=1e-12)
        np.testing.assert_allclose(X.col_norms_sq, np.einsum("ij,ij->j", base, base) + w, rtol=1e-14)
        b = rng.standard_normal(4)
        np.testing.assert_allclose(X.matvec(b), explicit @ b, rtol=1e-13)
        a = v.copy()
        X.axpy_col(2, 0.5, a)
        np.testing.assert_allclose(a, v + 0.5 * explicit[:, 2], rtol=1e-14)
        with pytest.raises(ValueError):
            X.normalized()


def _stacked_oracle(Xh, y, tail):
    """The reference's implicit-tail problem restated on the explicitly stacked
    design: tail rows after the base rows (so every sequential sum adds the tail
    term last, as _kernels.py does) and the reference norms base_sq + w (:56)."""
    Xh = Xh.toarray() if sp.issparse(Xh) else np.asarray(Xh, dtype=np.float64)
    p = Xh.shape[1]
    Xo = O.DesignMatrix(np.vstack([Xh, np.sqrt(tail) * np.eye(p)]))
    Xo.col_norms_sq = np.einsum("ij,ij->j", Xh, Xh) + tail
    Xo.col_norms = np.sqrt(Xo.col_norms_sq)
    return Xo, np.concatenate([y, np.zeros(p)])


@pytest.mark.parametrize("alpha,sparse", [(0.5, False), (0.3, True), (0.7, False)])
def test_elastic_net_tail_matches_oracle(alpha, sparse):
    """F2: to_lasso with a tail (elastic_net.py:34-46) solved on the device
    against the oracle on the stacked design, and the Elastic-Net KKT
    conditions (test_acceptance.py:331-348: kkt <= 1e-8 at epsilon 1e-10)."""
    c = synth.cfg0(p=400)
    Xh = sp.csc_matrix(np.where(np.abs(c.X) > 0.05, c.X, 0.0)) if sparse else c.X
    X = gs.DesignMatrix(Xh)
    lmax, _ = X.max_abs_correlation(c.y)
    en = gs.ElasticNetProblem(X, c.y, 0.15 * lmax / alpha, alpha)
    prob = gs.to_lasso(en)
    tail = (1.0 - alpha) * en.lam
    assert prob.X.tail_weight == tail and prob.y.size == X.n_base + X.n_cols
    cfg = gs.SolverConfig(epsilon=1e-10, max_passes=100_000)
    beta, cert, st = gs.solve(prob, cfg)
    assert st.converged and cert.gap <= 1e-10
    assert gs.kkt_residual(en, beta) <= 1e-8
    Xo, yo = _stacked_oracle(Xh, c.y, tail)
    b2, c2, st2 = O.solve(O.LassoProblem(Xo, yo, prob.lam), O.SolverConfig(epsilon=1e-10, max_passes=100_000))
    assert st.passes_done == st2.passes_done
    np.testing.assert_array_equal(beta != 0, b2 != 0)
    np.testing.assert_allclose(beta, b2, rtol=0, atol=1e-8 * max(1.0, float(np.max(np.abs(b2)))))
    assert abs(cert.gap - c2.gap) <= 1e-8 * max(abs(c2.primal), 1.0)
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "enet_cfg0_p400.npz"))
    k = [(0.5, False), (0.3, True), (0.7, False)].index((alpha, sparse))
    assert st.passes_done == int(g[f"c{k}_passes"])
    np.testing.assert_allclose(beta, g[f"c{k}_beta"], rtol=0, atol=1e-8 * max(1.0, float(np.max(np.abs(b2)))))


def test_elastic_net_path_and_report(tmp_path):
    """bench.py:153-182 per-lambda reduction, warm-started, on the device; and
    run_benchmark with l1_ratio < 1 (test_bench_cli.py:87-92)."""
    c = synth.cfg0(p=300)
    X = gs.DesignMatrix(c.X)
    lmax, _ = X.max_abs_correlation(c.y)
    grid = gs.lambda_grid(lmax, 6, 2.0)
    cfg = gs.SolverConfig(epsilon=1e-10, max_passes=100_000)
    res = gs.run_enet_path(X, c.y, grid, cfg, 0.5)
    assert res.converged.all()
    for t, lam in enumerate(grid):
        en = gs.ElasticNetProblem(X, c.y, float(lam) / 0.5, 0.5)
        assert gs.kkt_residual(en, res.betas[t]) <= 1e-8
    plain = gs.run_path(X, c.y, grid, cfg)
    same = gs.run_enet_path(X, c.y, grid, cfg, 1.0)
    assert np.array_equal(plain.betas, same.betas)
    from paper_1505_03410_b200.report import RunConfig, run_benchmark
    rep = run_benchmark(RunConfig(out_dir=str(tmp_path / "out"), rules=["gap_sphere"], epsilons=[1e-8],
                                  grid_T=5, grid_delta=2.0, l1_ratio=0.5), X, c.y)
    assert rep["summary"]["runs"][0]["n_converged"] == 5


@pytest.mark.parametrize("rule", ["gap_sphere", "gap_dome"])
def test_path_sparse_parallel_waves(rule):
    """CSC with rows plentiful relative to column length (n >= 256 x max column
    nnz, the cfg3 regime): the fully parallel waves (row map conflicts, parallel
    commit) against the oracle."""
    c = synth.cfg3(p=4000, n=4000, nnz_per_col=8)
    ra, rb, yy = _paths(c.X, c.y, 14, 2.0, c.epsilon, rule=rule)
    compare_paths(ra, rb, yy)
    assert np.all(ra.converged)


@pytest.mark.parametrize("n,mfac", [(40, "32"), (100, "32"), (200, "1"), (500, "32"), (1000, "32"), (1000, "1"),
                                    (1000, "1000")])
def test_path_blocked_chain_shapes(n, mfac, monkeypatch):
    """The blocked-chain consumer (GS_CD_GRAM=2) at every warp count it uses
    (n <= 128: 1 warp; 256: 2; 512: 4; 1024: 8), with a tight drift margin
    (GS_BLK_MFAC=1: windows end early and the next window is re-issued often)
    and a loose one, against the oracle."""
    monkeypatch.setenv("GS_CD_GRAM", "2")
    monkeypatch.setenv("GS_BLK_MFAC", mfac)
    c = synth.make_dense_case("blk", 7, n, 2500, 0.3, 40, "normal", 3.0, 12, 2.0, 1e-8)
    ra, rb, yy = _paths(c.X, c.y, 12, 2.0, c.epsilon)
    compare_paths(ra, rb, yy)
    if mfac == "1":
        assert sum(s.stats["cd_requeues"] for s in ra.states) > 0
