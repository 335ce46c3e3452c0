"""Host-facing DesignMatrix / problem / region methods on a CSC design of
non-trivial size, against the oracle (CSC ``matvec`` read its
output before the kernel finished on the B200; no GPU test covered it).

Reference: design_matrix.py:130-137 (matvec), problem.py:57-86
(primal_value with residual=None), regions.py:180-247 (ST3, inner radius).
"""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import gapsafe_oracle as O

pytestmark = pytest.mark.gpu
gs = pytest.importorskip("paper_1505_03410_b200")


def _case(seed=31, n=3000, p=5000, density=0.01, k=1500):
    rng = np.random.default_rng(seed)
    A = sp.random(n, p, density=density, format="csc", random_state=rng,
                  data_rvs=lambda m: rng.lognormal(0.0, 1.0, m))
    A.sort_indices()
    y = rng.standard_normal(n)
    beta = np.zeros(p)
    sup = rng.choice(p, k, replace=False)
    beta[sup] = rng.standard_normal(k)
    return A, y, beta


def _close(a, b, rtol=1e-12):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = max(1.0, float(np.max(np.abs(b))) if b.size else 1.0)
    assert np.max(np.abs(a - b)) <= rtol * scale, float(np.max(np.abs(a - b)))


@pytest.mark.parametrize("rep", range(3))
def test_csc_matvec_large(rep):
    A, _, beta = _case(seed=31 + rep)
    D = gs.DesignMatrix(A)
    ref = A @ beta
    for _ in range(4):                      # repeated calls: the race showed intermittently
        _close(D.matvec(beta), ref)


def test_csc_primal_value_residual_none():
    A, y, beta = _case()
    lam = 0.3 * float(np.max(np.abs(A.T @ y)))
    Po = O.LassoProblem(O.DesignMatrix(A), y, lam)
    P = gs.LassoProblem(gs.DesignMatrix(A), y, lam)
    assert gs.primal_value(P, beta) == pytest.approx(O.primal_value(Po, beta), rel=1e-12)
    rho = y - A @ beta
    assert gs.primal_value(P, beta, residual=rho) == pytest.approx(O.primal_value(Po, beta, residual=rho),
                                                                   rel=1e-13)


def test_csc_st3_and_inner_radius():
    A, y, beta = _case(seed=7)
    lam = 0.5 * float(np.max(np.abs(A.T @ y)))
    Xo, Xg = O.DesignMatrix(A), gs.DesignMatrix(A)
    Po, P = O.LassoProblem(Xo, y, lam), gs.LassoProblem(Xg, y, lam)
    rho = y - A @ beta
    tho = O.dual_scale(Po, rho)
    th = gs.dual_scale(P, rho)
    _close(th.theta, tho.theta, 1e-12)
    so, sg = O.region_st3(Po, tho), gs.region_st3(P, th)
    _close(sg.center, so.center, 1e-12)
    assert sg.radius == pytest.approx(so.radius, rel=1e-9, abs=1e-12)
    # inner radius of the gap dome with the residual recomputed on the device
    assert gs.inner_radius(P, beta) == pytest.approx(O.inner_radius(Po, beta), rel=1e-10, abs=1e-12)
    assert gs.inner_radius(P, beta, residual=rho) == pytest.approx(O.inner_radius(Po, beta, residual=rho),
                                                                   rel=1e-12, abs=1e-12)


def test_csc_transpose_dot_and_max_corr():
    A, y, _ = _case(seed=9)
    D = gs.DesignMatrix(A)
    _close(D.transpose_dot(y), A.T @ y)
    cols = np.arange(5, 5000, 7, dtype=np.int64)
    _close(D.transpose_dot(y, cols=cols), (A.T @ y)[cols])
    val, j = D.max_abs_correlation(y)
    c = np.abs(A.T @ y)
    assert j == int(np.argmax(c)) and val == pytest.approx(c.max(), rel=1e-13)


def test_dense_matvec_large():
    rng = np.random.default_rng(3)
    X = np.asfortranarray(rng.standard_normal((1500, 4000)))
    beta = np.zeros(4000)
    beta[rng.choice(4000, 900, replace=False)] = rng.standard_normal(900)
    D = gs.DesignMatrix(X)
    for _ in range(3):
        _close(D.matvec(beta), X @ beta)
