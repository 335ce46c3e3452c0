"""Parity on the BENCHMARKED workloads at their full sizes:
the first lambdas of the cfg1 path (the bench line's workload) and of the
cfg3 CSC path, with per-checkpoint active sets compared element by element
(track_active on both sides), against the oracle on the same seeded inputs.

Reference: path.py:52-105, solver.py:149-246."""

import numpy as np
import pytest

from oracle import gapsafe_oracle as O
from paper_1505_03410_b200 import synth
from parity import compare_paths

gs = pytest.importorskip("paper_1505_03410_b200")
pytestmark = pytest.mark.gpu


def _prefix_paths(case, k):
    X = gs.DesignMatrix(case.X)
    dev = gs.DeviceSolver(X, case.y)
    Xo = O.DesignMatrix(case.X)
    lmax, _ = Xo.max_abs_correlation(case.y)
    assert dev.lambda_max == pytest.approx(lmax, rel=1e-13)
    grid = O.lambda_grid(lmax, case.n_lambdas, case.delta)[:k]
    ra = gs.run_path(X, case.y, grid, gs.SolverConfig(epsilon=case.epsilon, max_passes=100_000,
                                                      track_active=True), solver=dev)
    rb = O.run_path(Xo, case.y, grid, O.SolverConfig(epsilon=case.epsilon, max_passes=100_000,
                                                     track_active=True), cache_lambda_max=True)
    return ra, rb, float(case.y @ case.y)


def test_cfg1_full_size_first_64_lambdas():
    """configs[1] at full size (1000 x 100,000 f64): the first 64 of its 100
    lambdas, every checkpoint's active set identical."""
    c = synth.cfg1()
    ra, rb, yy = _prefix_paths(c, 64)
    compare_paths(ra, rb, yy)
    assert sum(len(s.active_history) for s in ra.states) > 100


def test_cfg3_full_size_first_10_lambdas():
    """configs[3] at full size (CSC 20,000 x 1,000,000, 20 nnz per column):
    the first 10 lambdas."""
    c = synth.cfg3()
    ra, rb, yy = _prefix_paths(c, 10)
    compare_paths(ra, rb, yy)
