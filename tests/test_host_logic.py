"""Host-side logic that needs no GPU: config validation, value types, the
lambda grid, scalar identities, and the seeded generators."""

import numpy as np
import pytest

import paper_1505_03410_b200 as gs
from paper_1505_03410_b200 import synth


def test_solver_config_validation():
    """pkg/tests/test_solver.py:249-260."""
    with pytest.raises(ValueError):
        gs.SolverConfig(epsilon=0.0)
    with pytest.raises(ValueError):
        gs.SolverConfig(screen_every=0)
    with pytest.raises(ValueError):
        gs.SolverConfig(max_passes=0)
    with pytest.raises(ValueError):
        gs.SolverConfig(rule="banana")
    assert gs.SolverConfig(rule="gap_dome").rule is gs.Rule.GAP_DOME
    assert gs.SolverConfig().rule is gs.Rule.GAP_SPHERE


def test_soft_threshold_hand_values():
    """pkg/tests/test_solver.py:63-84."""
    assert gs.soft_threshold(1.0, 3.0) == 2.0
    assert gs.soft_threshold(1.0, -3.0) == -2.0
    assert gs.soft_threshold(1.0, 0.5) == 0.0
    assert gs.soft_threshold(2.0, 2.0) == 0.0
    with pytest.raises(ValueError):
        gs.soft_threshold(-0.1, 1.0)


def test_lambda_grid():
    """pkg/tests/test_problem.py:149-168."""
    np.testing.assert_allclose(gs.lambda_grid(2.0, 4, 3.0), [2.0, 0.2, 0.02, 0.002], rtol=1e-14)
    g = gs.lambda_grid(1.0, 100, 3.0)
    assert g.size == 100 and g[0] == 1.0 and g[-1] == pytest.approx(1e-3)
    with pytest.raises(ValueError):
        gs.lambda_grid(1.0, 1, 3.0)


def test_sequential_radius_sq_hand_values():
    """pkg/tests/test_path.py:272-295."""
    assert gs.sequential_radius_sq(4.0, 2.0, 1.0, 9.0, 0.5) == 12.0
    assert gs.sequential_radius_sq(9.0, 3.0, 1.0, 36.0, 6.75) == 37.5
    assert gs.sequential_radius_sq(7.0, 2.0, 2.0, 5.0, 1.0) == 7.0
    with pytest.raises(ValueError):
        gs.sequential_radius_sq(1.0, 1.0, 2.0, 1.0, 1.0)


def test_sphere_validation():
    with pytest.raises(ValueError):
        gs.Sphere(center=np.zeros(2), radius=-1.0)
    with pytest.raises(ValueError):
        gs.Sphere(center=np.zeros(2), radius=np.inf)


def test_generators_deterministic_and_normalised():
    a, b = synth.cfg0(p=300), synth.cfg0(p=300)
    assert np.array_equal(a.X, b.X) and np.array_equal(a.y, b.y)
    assert a.X.flags.f_contiguous
    np.testing.assert_allclose(np.linalg.norm(a.X, axis=0), 1.0, rtol=1e-12)
    np.testing.assert_allclose(a.X.mean(axis=0), 0.0, atol=1e-15)
    assert np.count_nonzero(a.beta_star) == 20
    sig = a.X @ a.beta_star
    assert np.linalg.norm(sig) / np.linalg.norm(a.y - sig) == pytest.approx(3.0, rel=1e-12)
    c3 = synth.cfg3(p=5000, n=300, nnz_per_col=20)
    assert c3.X.has_sorted_indices and np.all(np.diff(c3.X.indptr) == 20)
    rows = c3.X.indices.reshape(5000, 20)
    assert np.all(np.diff(rows, axis=1) > 0)          # distinct, sorted rows per column
    np.testing.assert_allclose(np.sqrt(np.asarray(c3.X.multiply(c3.X).sum(0)).ravel()), 1.0, rtol=1e-12)
    assert np.array_equal(synth.cfg4_rows(3), synth.cfg4_rows(3))
