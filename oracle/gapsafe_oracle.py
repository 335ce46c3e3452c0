"""CPU oracle for the Gap Safe Lasso path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product (``paper_1505_03410_b200``) never does: it runs on the GPU or fails.

This is a restatement of the reference's hot path
(/root/reference/pkg/src/gapsafe/{design_matrix,problem,regions,solver,path}.py)
with the same numpy/BLAS calls in the same order, and with the numba column
kernels replaced by the plain-C restatement in ``oracle/kernels.c``
(sequential, non-FMA -- bit-identical to the numba kernels).  On one machine
it therefore reproduces the reference bit-for-bit; ``tests/golden/`` holds
reference outputs (made by ``tests/golden/make_golden.py`` with the real
reference imported) and ``tests/test_oracle_golden.py`` pins this module to
them.  Parity pin status: pinned (golden vectors + direct comparison with
the reference where it is importable).

Scope: the north_star path with every screening rule of the reference
(``none``, ``static``, ``dynamic``, ``st3``, ``gap_sphere``, ``gap_dome``;
regions.py:23-273, solver.py:104-126); Elastic-Net and I/O are out of scope
(SURVEY.md §2).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_kernels.so")
_lib = None

_f64p = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build_kernels(force: bool = False) -> str:
    """Compile oracle/kernels.c into oracle/liboracle_kernels.so (gcc)."""
    src = os.path.join(_HERE, "kernels.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        import subprocess
        subprocess.check_call(
            ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
             "-fno-fast-math", "-o", _LIB_PATH, src])
    return _LIB_PATH


def _kernels():
    global _lib
    if _lib is None:
        build_kernels()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_tdot_dense.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, _f64p,
                                          _i64p, ctypes.c_int64, ctypes.c_double, _f64p]
        lib.oracle_tdot_csc.argtypes = [_f64p, _i32p, _i32p, ctypes.c_int64, _f64p,
                                        _i64p, ctypes.c_int64, ctypes.c_double, _f64p]
        lib.oracle_cd_pass_dense.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, _f64p,
                                             _f64p, _i64p, ctypes.c_int64, ctypes.c_double,
                                             _f64p, ctypes.c_double]
        lib.oracle_cd_pass_csc.argtypes = [_f64p, _i32p, _i32p, ctypes.c_int64, _f64p,
                                           _f64p, _i64p, ctypes.c_int64, ctypes.c_double,
                                           _f64p, ctypes.c_double]
        for name in ("oracle_tdot_dense", "oracle_tdot_csc",
                     "oracle_cd_pass_dense", "oracle_cd_pass_csc"):
            getattr(lib, name).restype = None
        _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# kernel-level entry points (same signatures as _kernels.py)
# ---------------------------------------------------------------------------

def tdot_dense(X, v, cols, tail_scale, out):
    """_kernels.py:14-24."""
    assert X.flags.f_contiguous and X.dtype == np.float64
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    _kernels().oracle_tdot_dense(_p(X, _f64p), X.shape[0], X.shape[0], _p(v, _f64p),
                                 _p(cols, _i64p), cols.size, float(tail_scale),
                                 _p(out, _f64p))


def tdot_csc(data, indices, indptr, n_base, v, cols, tail_scale, out):
    """_kernels.py:27-36."""
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    _kernels().oracle_tdot_csc(_p(data, _f64p), _p(indices, _i32p), _p(indptr, _i32p),
                               int(n_base), _p(v, _f64p), _p(cols, _i64p), cols.size,
                               float(tail_scale), _p(out, _f64p))


def cd_pass_dense(X, beta, rho, active, lam, norms_sq, tail_scale):
    """_kernels.py:39-64 (beta, rho updated in place)."""
    assert X.flags.f_contiguous and X.dtype == np.float64
    active = np.ascontiguousarray(active, dtype=np.int64)
    _kernels().oracle_cd_pass_dense(_p(X, _f64p), X.shape[0], X.shape[0],
                                    _p(beta, _f64p), _p(rho, _f64p), _p(active, _i64p),
                                    active.size, float(lam), _p(norms_sq, _f64p),
                                    float(tail_scale))


def cd_pass_csc(data, indices, indptr, n_base, beta, rho, active, lam, norms_sq,
                tail_scale):
    """_kernels.py:67-92 (beta, rho updated in place)."""
    active = np.ascontiguousarray(active, dtype=np.int64)
    _kernels().oracle_cd_pass_csc(_p(data, _f64p), _p(indices, _i32p), _p(indptr, _i32p),
                                  int(n_base), _p(beta, _f64p), _p(rho, _f64p),
                                  _p(active, _i64p), active.size, float(lam),
                                  _p(norms_sq, _f64p), float(tail_scale))


# ---------------------------------------------------------------------------
# DesignMatrix (design_matrix.py:22-187, pure-Lasso subset: tail_weight = 0)
# ---------------------------------------------------------------------------

class DesignMatrix:
    """design_matrix.py:34-57: dense -> F-order f64, sparse -> canonical CSC."""

    def __init__(self, storage):
        if sp.issparse(storage):
            mat = sp.csc_matrix(storage).astype(np.float64)
            mat.sum_duplicates()
            mat.sort_indices()
            self._mat = mat
            self.is_sparse = True
            base_sq = np.asarray(mat.multiply(mat).sum(axis=0)).ravel()
        else:
            arr = np.asfortranarray(np.asarray(storage, dtype=np.float64))
            self._mat = arr
            self.is_sparse = False
            base_sq = np.einsum("ij,ij->j", arr, arr)         # design_matrix.py:50
        self.n_base, self.n_cols = self._mat.shape
        self.n_rows = self.n_base
        self.col_norms_sq = base_sq + 0.0                      # :56 (tail_weight 0)
        self.col_norms = np.sqrt(self.col_norms_sq)            # :57

    def axpy_col(self, j, a, v):
        """design_matrix.py:115-128."""
        if a == 0.0:
            return
        if self.is_sparse:
            lo, hi = self._mat.indptr[j], self._mat.indptr[j + 1]
            v[self._mat.indices[lo:hi]] += a * self._mat.data[lo:hi]
        else:
            v[: self.n_base] += a * self._mat[:, j]

    def col_dot(self, j, v):
        """design_matrix.py:100-113 (no implicit tail in the oracle)."""
        v = np.asarray(v, dtype=np.float64)
        if self.is_sparse:
            lo, hi = self._mat.indptr[j], self._mat.indptr[j + 1]
            return float(np.dot(self._mat.data[lo:hi], v[self._mat.indices[lo:hi]]))
        return float(np.dot(self._mat[:, j], v[: self.n_base]))

    def matvec(self, beta):
        """design_matrix.py:130-137."""
        beta = np.asarray(beta, dtype=np.float64)
        return np.asarray(self._mat @ beta).ravel()

    def transpose_dot(self, v, cols=None):
        """design_matrix.py:139-158."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        if cols is None:
            return np.asarray(self._mat.T @ v[: self.n_base]).ravel().astype(
                np.float64, copy=False)
        cols = np.asarray(cols, dtype=np.int64)
        out = np.empty(cols.size, dtype=np.float64)
        if self.is_sparse:
            m = self._mat
            tdot_csc(m.data, m.indices, m.indptr, self.n_base, v, cols, 0.0, out)
        else:
            tdot_dense(self._mat, v, cols, 0.0, out)
        return out

    def max_abs_correlation(self, v, restrict=None):
        """design_matrix.py:160-174 (ties -> smallest index)."""
        if restrict is not None:
            restrict = np.asarray(restrict, dtype=np.int64)
            if restrict.size == 0:
                raise ValueError("empty restriction set")
        dots = np.abs(self.transpose_dot(v, cols=restrict))
        i = int(np.argmax(dots))
        j = i if restrict is None else int(restrict[i])
        return float(dots[i]), j

    def run_pass(self, beta, rho, active, lam):
        """solver.py:93-101 _run_pass."""
        if self.is_sparse:
            m = self._mat
            cd_pass_csc(m.data, m.indices, m.indptr, self.n_base, beta, rho, active,
                        lam, self.col_norms_sq, 0.0)
        else:
            cd_pass_dense(self._mat, beta, rho, active, lam, self.col_norms_sq, 0.0)


# ---------------------------------------------------------------------------
# problem.py
# ---------------------------------------------------------------------------

class InfeasibleDualError(ValueError):
    pass


class NumericalInconsistencyError(RuntimeError):
    pass


@dataclass(frozen=True)
class DualPoint:
    theta: np.ndarray
    feasibility_margin: float
    interpolating: bool = False


@dataclass(frozen=True)
class GapCertificate:
    primal: float
    dual: float
    gap: float


class LassoProblem:
    """problem.py:41-54.  ``lambda_max`` may be passed in to skip the
    redundant full X^T y pass (it is deterministic, hence identical)."""

    def __init__(self, X, y, lam, lambda_max=None):
        y = np.ascontiguousarray(y, dtype=np.float64)
        if lam <= 0:
            raise ValueError("lambda must be positive")
        self.X, self.y, self.lam = X, y, float(lam)
        if lambda_max is None:
            self.lambda_max, self.j_star = X.max_abs_correlation(y)
        else:
            self.lambda_max, self.j_star = lambda_max
        if self.lam > self.lambda_max * (1 + 1e-12):
            raise ValueError(f"lambda={lam} exceeds lambda_max={self.lambda_max}")
        self.y_norm_sq = float(np.dot(y, y))


def primal_value(prob, beta, residual=None):
    """problem.py:57-69."""
    beta = np.asarray(beta, dtype=np.float64)
    if residual is None:
        residual = prob.y - prob.X.matvec(beta)
    return 0.5 * float(np.dot(residual, residual)) \
        + prob.lam * float(np.sum(np.abs(beta)))


def dual_value(prob, theta):
    """problem.py:72-78."""
    if theta.feasibility_margin < -1e-9:
        raise InfeasibleDualError(f"dual point infeasible: margin={theta.feasibility_margin}")
    diff = theta.theta - prob.y / prob.lam
    return 0.5 * prob.y_norm_sq - 0.5 * prob.lam ** 2 * float(np.dot(diff, diff))


def duality_gap(prob, beta, theta, residual=None):
    """problem.py:81-86."""
    p = primal_value(prob, beta, residual=residual)
    d = dual_value(prob, theta)
    return GapCertificate(primal=p, dual=d, gap=p - d)


def dual_scale(prob, residual, restrict=None):
    """problem.py:98-123 (Eq. 10 clip form)."""
    rho = np.ascontiguousarray(residual, dtype=np.float64)
    rho_sq = float(np.dot(rho, rho))
    if rho_sq == 0.0:
        return DualPoint(theta=np.zeros_like(rho), feasibility_margin=1.0,
                         interpolating=True)
    corr, _ = prob.X.max_abs_correlation(rho, restrict=restrict)
    raw = float(np.dot(prob.y, rho)) / (prob.lam * rho_sq)
    if corr > 0.0:
        bound = 1.0 / corr
        alpha = min(max(raw, -bound), bound)
    else:
        alpha = raw
    theta = alpha * rho
    return DualPoint(theta=theta, feasibility_margin=1.0 - abs(alpha) * corr)


def lambda_grid(lambda_max, T, delta):
    """problem.py:126-133."""
    if T < 2:
        raise ValueError("T must be at least 2")
    if delta <= 0:
        raise ValueError("delta must be positive")
    t = np.arange(T)
    return lambda_max * 10.0 ** (-delta * t / (T - 1))


# ---------------------------------------------------------------------------
# regions.py (gap sphere only)
# ---------------------------------------------------------------------------

SCREEN_SAFETY = 1e-9        # regions.py:126


@dataclass(frozen=True)
class Sphere:
    center: np.ndarray
    radius: float


@dataclass(frozen=True)
class Dome:
    """regions.py:35-57: B(c, r) & {theta : n^T theta <= n^T c - ratio r}."""
    center: np.ndarray
    radius: float
    ratio: float
    normal: np.ndarray


@dataclass(frozen=True)
class ScreenResult:
    zero_set: np.ndarray
    active_set: np.ndarray
    mu: np.ndarray


def _sphere_mu_values(s, X, cols):
    """regions.py:75-79."""
    ct = X.transpose_dot(s.center, cols=cols)
    norms = X.col_norms if cols is None else X.col_norms[cols]
    return np.abs(ct) + s.radius * norms


def _dome_mu_values(d, X, cols):
    """regions.py:82-97."""
    ct = X.transpose_dot(d.center, cols=cols)
    nt = X.transpose_dot(d.normal, cols=cols)
    norms = X.col_norms if cols is None else X.col_norms[cols]
    r, a = d.radius, min(max(d.ratio, -1.0), 1.0)
    cross = r * np.sqrt(np.maximum(norms ** 2 - nt ** 2, 0.0) * (1.0 - a ** 2))
    sig_pos = np.where(nt < -a * norms, ct + r * norms, ct - r * a * nt + cross)
    sig_neg = np.where(-nt < -a * norms, -ct + r * norms, -ct + r * a * nt + cross)
    return np.maximum(sig_pos, sig_neg)


def mu_values(region, X, cols=None):
    """regions.py:100-107."""
    if isinstance(region, Sphere):
        return _sphere_mu_values(region, X, cols)
    if isinstance(region, Dome):
        return _dome_mu_values(region, X, cols)
    raise TypeError(f"unknown region type: {type(region)!r}")


def screen(region, X, tol=SCREEN_SAFETY, cols=None):
    """regions.py:129-139."""
    mus = mu_values(region, X, cols=cols)
    idx = np.arange(X.n_cols) if cols is None else np.asarray(cols)
    zero = mus < 1.0 - tol
    return ScreenResult(zero_set=idx[zero], active_set=idx[~zero], mu=mus)


def gap_radius(prob, gap):
    """regions.py:213-218."""
    if gap < -1e-10:
        raise NumericalInconsistencyError(f"negative duality gap beyond tolerance: {gap}")
    return float(np.sqrt(2.0 * max(gap, 0.0)) / prob.lam)


def region_gap_sphere(prob, beta, theta, residual=None, gap=None):
    """regions.py:221-232."""
    if gap is None:
        gap = duality_gap(prob, beta, theta, residual=residual).gap
    return Sphere(center=np.array(theta.theta, dtype=np.float64),
                  radius=gap_radius(prob, gap))


def region_static(prob):
    """regions.py:162-165."""
    r = abs(1.0 / prob.lam - 1.0 / prob.lambda_max) * np.sqrt(prob.y_norm_sq)
    return Sphere(center=prob.y / prob.lam, radius=float(r))


def region_dynamic(prob, theta):
    """regions.py:168-174."""
    if theta.feasibility_margin < -1e-9:
        raise ValueError("theta must be dual feasible")
    center = prob.y / prob.lam
    return Sphere(center=center, radius=float(np.linalg.norm(theta.theta - center)))


def region_st3(prob, theta):
    """regions.py:177-197."""
    if theta.feasibility_margin < -1e-9:
        raise ValueError("theta must be dual feasible")
    center = prob.y / prob.lam
    big_r = float(np.linalg.norm(theta.theta - center))
    xj = np.zeros(prob.X.n_cols)
    xj[prob.j_star] = 1.0
    col = prob.X.matvec(xj)
    sgn = np.sign(prob.X.col_dot(prob.j_star, prob.y)) or 1.0
    norm_j = prob.X.col_norms[prob.j_star]
    dist = (prob.lambda_max / prob.lam - 1.0) / norm_j
    radicand = big_r ** 2 - dist ** 2
    if radicand < 0:
        radicand = 0.0
    new_center = center - (dist / norm_j) * sgn * col
    return Sphere(center=new_center, radius=float(np.sqrt(radicand)))


def inner_radius(prob, beta, residual=None):
    """regions.py:235-247."""
    beta = np.asarray(beta, dtype=np.float64)
    if residual is None:
        residual = prob.y - prob.X.matvec(beta)
    val = prob.y_norm_sq - float(np.dot(residual, residual)) - 2.0 * prob.lam * float(np.sum(np.abs(beta)))
    return float(np.sqrt(max(val, 0.0))) / prob.lam


def region_gap_dome(prob, beta, theta, residual=None):
    """regions.py:250-273."""
    if theta.feasibility_margin < -1e-9:
        raise ValueError("theta must be dual feasible")
    yl = prob.y / prob.lam
    diff = yl - theta.theta
    big_r = float(np.linalg.norm(diff))
    if big_r == 0.0:
        return Sphere(center=np.array(theta.theta), radius=0.0)
    r_in = inner_radius(prob, beta, residual=residual)
    if r_in > big_r * (1 + 1e-9) + 1e-12:
        raise NumericalInconsistencyError(f"inner radius {r_in} exceeds outer radius {big_r}")
    r_in = min(r_in, big_r)
    ratio = 2.0 * (r_in / big_r) ** 2 - 1.0
    return Dome(center=0.5 * (yl + theta.theta), radius=0.5 * big_r, ratio=ratio, normal=diff / big_r)


def _make_region(rule, prob, beta, theta, rho, gap):
    """solver.py:104-119."""
    if rule == "none":
        return None
    if rule == "static":
        return region_static(prob)
    if rule == "dynamic":
        return region_dynamic(prob, theta)
    if rule == "st3":
        return region_st3(prob, theta)
    if rule == "gap_sphere":
        return region_gap_sphere(prob, beta, theta, gap=gap)
    if rule == "gap_dome":
        return region_gap_dome(prob, beta, theta, residual=rho)
    raise ValueError(f"unknown rule {rule}")


def _trace_radius(rule, region, prob, gap):
    """solver.py:122-126."""
    if rule in ("none", "gap_sphere", "gap_dome"):
        return gap_radius(prob, max(gap, 0.0))
    return region.radius if region is not None else float("nan")


# ---------------------------------------------------------------------------
# solver.py
# ---------------------------------------------------------------------------

@dataclass
class SolverConfig:
    epsilon: float = 1e-8
    max_passes: int = 10_000
    screen_every: int = 10
    rule: str = "gap_sphere"
    track_active: bool = False
    on_checkpoint: object = None

    def __post_init__(self):
        self.rule = getattr(self.rule, "value", self.rule)
        if self.rule not in ("none", "static", "dynamic", "st3", "gap_sphere", "gap_dome"):
            raise ValueError(f"unknown rule {self.rule}")


@dataclass
class SolverState:
    beta: np.ndarray
    residual: np.ndarray
    active: np.ndarray
    theta: DualPoint | None
    cert: GapCertificate | None
    passes_done: int
    converged: bool
    screen_trace: list = field(default_factory=list)
    active_history: list = field(default_factory=list)


def _solve_at_lambda_max(prob, config):
    """solver.py:129-146."""
    beta = np.zeros(prob.X.n_cols)
    theta = DualPoint(theta=prob.y / prob.lam, feasibility_margin=0.0)
    cert = GapCertificate(primal=0.5 * prob.y_norm_sq, dual=0.5 * prob.y_norm_sq, gap=0.0)
    if config.rule == "none":
        active = np.flatnonzero(prob.X.col_norms > 0)
    else:
        mus = np.abs(prob.X.transpose_dot(theta.theta))
        active = np.flatnonzero(mus >= 1.0 - SCREEN_SAFETY)
    state = SolverState(beta=beta, residual=prob.y.copy(), active=active, theta=theta,
                        cert=cert, passes_done=0, converged=True)
    state.screen_trace.append((0, active.size, 0.0, 0.0))
    if config.track_active:
        state.active_history.append(active.copy())
    if config.on_checkpoint is not None:
        config.on_checkpoint(active)
    return beta, cert, state


def solve(prob, config, warm_beta=None, active0=None):
    """solver.py:149-246 (Algorithm 1)."""
    X, lam = prob.X, prob.lam
    if lam >= prob.lambda_max * (1 - 1e-14):
        return _solve_at_lambda_max(prob, config)
    p = X.n_cols
    beta = np.zeros(p) if warm_beta is None else np.array(warm_beta, dtype=np.float64)
    if active0 is None:
        active = np.flatnonzero(X.col_norms > 0)
    else:
        active = np.asarray(active0, dtype=np.int64)
        active = active[X.col_norms[active] > 0]
    mask = np.zeros(p, dtype=bool)
    mask[active] = True
    beta[~mask] = 0.0
    rho = prob.y - X.matvec(beta)
    state = SolverState(beta=beta, residual=rho, active=active, theta=None, cert=None,
                        passes_done=0, converged=False)
    f = config.screen_every
    for k in range(1, config.max_passes + 1):
        if f == 1 or k % f == 1:
            rho = prob.y - X.matvec(beta)
            state.residual = rho
            if state.active.size == 0:
                theta = dual_scale(prob, rho)
                cert = duality_gap(prob, beta, theta, residual=rho)
                state.theta, state.cert = theta, cert
                state.converged = cert.gap <= config.epsilon
                state.screen_trace.append((state.passes_done, 0, cert.gap,
                                           gap_radius(prob, max(cert.gap, 0.0))))
                if config.track_active:
                    state.active_history.append(state.active.copy())
                if config.on_checkpoint is not None:
                    config.on_checkpoint(state.active)
                break
            theta = dual_scale(prob, rho, restrict=state.active)
            pre_gap = duality_gap(prob, beta, theta, residual=rho).gap
            region = _make_region(config.rule, prob, beta, theta, rho, pre_gap)
            if region is not None:
                mus = mu_values(region, X, cols=state.active)
                keep = mus >= 1.0 - SCREEN_SAFETY
                dropped = state.active[~keep]
                if dropped.size:
                    for j in dropped:
                        if beta[j] != 0.0:
                            X.axpy_col(j, beta[j], rho)
                            beta[j] = 0.0
                    state.active = state.active[keep]
            cert = duality_gap(prob, beta, theta, residual=rho)
            state.theta, state.cert = theta, cert
            state.screen_trace.append((state.passes_done, state.active.size, cert.gap,
                                       _trace_radius(config.rule, region, prob, cert.gap)))
            if config.track_active:
                state.active_history.append(state.active.copy())
            if config.on_checkpoint is not None:
                config.on_checkpoint(state.active)
            if cert.gap <= config.epsilon:
                state.converged = True
                break
            if state.active.size == 0:
                break
        elif k % 100 == 0:
            rho = prob.y - X.matvec(beta)
            state.residual = rho
        X.run_pass(beta, rho, state.active, lam)
        state.passes_done += 1
    if not state.converged:
        rho = prob.y - X.matvec(beta)
        state.residual = rho
        theta = dual_scale(prob, rho, restrict=state.active if state.active.size else None)
        state.theta = theta
        state.cert = duality_gap(prob, beta, theta, residual=rho)
        state.converged = state.cert.gap <= config.epsilon
    return beta, state.cert, state


# ---------------------------------------------------------------------------
# path.py
# ---------------------------------------------------------------------------

@dataclass
class PathResult:
    lambdas: np.ndarray
    betas: np.ndarray
    certs: list
    traces: list
    timings: list
    converged: np.ndarray
    states: list = field(default_factory=list)


def run_path(X, y, grid, config, cache_lambda_max=False, max_points=None, time_budget_s=None):
    """path.py:52-105.

    ``cache_lambda_max`` skips the identical per-lambda X^T y pass
    (problem.py:50); ``max_points`` stops after that many grid points and
    ``time_budget_s`` after the point at which the cumulative per-lambda time
    exceeds the budget (the bounded CPU-baseline sample).  The defaults give
    the reference behaviour.
    """
    grid = np.asarray(grid, dtype=np.float64)
    if grid.size == 0:
        raise ValueError("empty lambda grid")
    if np.any(np.diff(grid) > 0):
        raise ValueError("grid must be non-increasing")
    T = grid.size if max_points is None else min(grid.size, int(max_points))
    p = X.n_cols
    betas = np.zeros((T, p))
    certs, traces, timings, states = [], [], [], []
    conv = np.zeros(T, dtype=bool)
    prev_beta = prev_theta = prev_resid = None
    lmax = X.max_abs_correlation(np.ascontiguousarray(y, dtype=np.float64)) \
        if cache_lambda_max else None
    for t in range(T):
        lam = grid[t]
        t0 = time.perf_counter()
        prob = LassoProblem(X, y, lam, lambda_max=lmax)
        warm = None if prev_beta is None else prev_beta
        active0 = None
        if (prev_theta is not None and not prev_theta.interpolating
                and config.rule in ("gap_sphere", "gap_dome")):
            if config.rule == "gap_sphere":
                region = region_gap_sphere(prob, prev_beta, prev_theta, residual=prev_resid)
            else:
                region = region_gap_dome(prob, prev_beta, prev_theta, residual=prev_resid)
            active0 = screen(region, X).active_set
        beta, cert, state = solve(prob, config, warm_beta=warm, active0=active0)
        timings.append(time.perf_counter() - t0)
        betas[t] = beta
        certs.append(cert)
        traces.append(state.screen_trace)
        states.append(state)
        conv[t] = state.converged
        prev_beta, prev_theta, prev_resid = beta, state.theta, state.residual
        if time_budget_s is not None and sum(timings) >= time_budget_s:
            T = t + 1
            break
    return PathResult(lambdas=grid[:T], betas=betas[:T], certs=certs, traces=traces,
                      timings=timings, converged=conv[:T], states=states)
