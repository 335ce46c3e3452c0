"""Coordinate descent with interlaced Gap Safe screening (drop-in for
gapsafe.solver, /root/reference/pkg/src/gapsafe/solver.py:1-246).

``solve`` runs Algorithm 1 on the device: residual resync, Eq. 10 dual point
with the restricted infinity norm, pre-drop gap, sphere test, drop axpys,
post-drop certificate and trace at every checkpoint, and the CD epochs in
between (one CTA per problem, exact certified-zero skipping).  The host only
sequences launches and reads one scalar block per checkpoint.

Rules on the GPU: every ``Rule`` of the reference (solver.py:24-32, 104-126).
``gap_sphere`` is the north_star path; ``static``, ``dynamic``, ``st3`` and
``gap_dome`` reuse the same checkpoint with their own
per-column test, evaluated from q = X^T y (cached at solver creation),
X^T x_jstar (ST3, built on first use) and the restricted dots X_A^T rho --
no extra pass over the design.  Batched problems (cfg4) run ``none`` /
``gap_sphere``.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .problem import DualPoint, GapCertificate, LassoProblem


class Rule(str, enum.Enum):
    """Screening rule used at solver checkpoints (solver.py:24-32)."""

    NONE = "none"
    STATIC = "static"
    DYNAMIC = "dynamic"
    ST3 = "st3"
    GAP_SPHERE = "gap_sphere"
    GAP_DOME = "gap_dome"


_GPU_RULES = {Rule.NONE: _lib.GS_RULE_NONE, Rule.GAP_SPHERE: _lib.GS_RULE_GAP_SPHERE,
              Rule.STATIC: _lib.GS_RULE_STATIC, Rule.DYNAMIC: _lib.GS_RULE_DYNAMIC,
              Rule.ST3: _lib.GS_RULE_ST3, Rule.GAP_DOME: _lib.GS_RULE_GAP_DOME}
# batched problems (cfg4) run the north_star rules only
_BATCH_RULES = {Rule.NONE: _lib.GS_RULE_NONE, Rule.GAP_SPHERE: _lib.GS_RULE_GAP_SPHERE}


@dataclass
class SolverConfig:
    """solver.py:35-54 (same fields, defaults and validation)."""

    epsilon: float = 1e-8
    max_passes: int = 10_000
    screen_every: int = 10
    rule: Rule = Rule.GAP_SPHERE
    track_active: bool = False
    on_checkpoint: object = None
    # B200 extra: exact certified-zero skipping inside the CD epoch
    certify: bool = True

    def __post_init__(self):
        self.rule = Rule(self.rule)
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.screen_every < 1:
            raise ValueError("screen_every must be at least 1")
        if self.max_passes < 1:
            raise ValueError("max_passes must be at least 1")


@dataclass
class SolverState:
    """solver.py:57-68."""

    beta: np.ndarray
    residual: np.ndarray
    active: np.ndarray
    theta: DualPoint | None
    cert: GapCertificate | None
    passes_done: int
    converged: bool
    screen_trace: list = field(default_factory=list)
    active_history: list = field(default_factory=list)
    # B200 extras: CD work counters and device time of the solve
    stats: dict = field(default_factory=dict)


def soft_threshold(u: float, x: float) -> float:
    """sign(x) (|x| - u)_+ (solver.py:71-79)."""
    if u < 0:
        raise ValueError("threshold must be non-negative")
    if x > u:
        return x - u
    if x < -u:
        return x + u
    return 0.0


def cd_pass(state: SolverState, prob: LassoProblem, order: np.ndarray | None = None,
            exact_order: bool = False) -> SolverState:
    """One cyclic CD pass over the active set, in place (solver.py:82-90).

    ``exact_order`` runs the reference's sequential non-FMA arithmetic
    (bit-exact with _kernels.cd_pass_*); otherwise the production kernel."""
    active = state.active if order is None else np.asarray(order, dtype=np.int64)
    active = np.ascontiguousarray(active, dtype=np.int64)
    X = prob.X
    if np.any(X.col_norms[active] == 0.0):
        raise RuntimeError("zero-norm column in active set")
    beta = np.ascontiguousarray(state.beta, dtype=np.float64)
    rho = np.ascontiguousarray(state.residual, dtype=np.float64)
    _lib.check(X._lib.gs_cd_pass(X.handle, _lib.f64p(beta), _lib.f64p(rho), _lib.i64p(active),
                                 active.size, float(prob.lam), None, 0.0, int(exact_order)))
    if beta is not state.beta:
        state.beta[...] = beta
    if rho is not state.residual:
        state.residual[...] = rho
    state.passes_done += 1
    return state


class DeviceSolver:
    """One device solver handle for a fixed (X, y): y, beta, rho, theta and
    the active set stay resident in HBM across solves (warm starts and the
    sequential screen of run_path never cross PCIe)."""

    def __init__(self, X, y: np.ndarray):
        self.X = X
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        if self.y.shape != (X.n_rows,):
            raise ValueError(f"y has length {self.y.shape}, expected ({X.n_rows},)")
        self._lib = X._lib
        h = ctypes.c_void_p()
        _lib.check(self._lib.gs_solver_create(X.handle, _lib.f64p(self.y), ctypes.byref(h)))
        self._h = h
        lm, js, yn = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _lib.check(self._lib.gs_solver_lambda_max(h, ctypes.byref(lm), ctypes.byref(js), ctypes.byref(yn)))
        self.lambda_max, self.j_star, self.y_norm_sq = lm.value, js.value, yn.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.gs_solver_free(h)
            self._h = None

    def set_lambda_max(self, lambda_max: float) -> None:
        """Use the whole problem's lambda_max (sharded paths solve on a
        gathered column subset; problem.py:50)."""
        _lib.check(self._lib.gs_solver_set_lambda_max(self._h, float(lambda_max)))
        self.lambda_max = float(lambda_max)

    def set_beta(self, beta):
        if beta is None:
            _lib.check(self._lib.gs_solver_set_beta(self._h, None))
        else:
            b = np.ascontiguousarray(beta, dtype=np.float64)
            if b.shape != (self.X.n_cols,):
                raise ValueError("warm_beta has wrong length")
            _lib.check(self._lib.gs_solver_set_beta(self._h, _lib.f64p(b)))

    def seq_screen(self, lam: float) -> int:
        cnt = ctypes.c_int64()
        _lib.check(self._lib.gs_solver_seq_screen(self._h, float(lam), ctypes.byref(cnt)))
        return cnt.value

    def solve(self, lam: float, config: SolverConfig, active0=None, active0_mode: int = 0,
              beta_out: np.ndarray | None = None):
        """Run solver.py:149-246 on the device; returns (beta, cert, state)."""
        if config.rule not in _GPU_RULES:
            raise NotImplementedError(
                f"rule {config.rule.value!r} is not on the B200 path in this build "
                f"(supported: {', '.join(r.value for r in _GPU_RULES)})")
        X = self.X
        n, p = X.n_rows, X.n_cols
        cap = config.max_passes // config.screen_every + 4
        beta = np.empty(p) if beta_out is None else beta_out
        rho = np.empty(n)
        theta = np.empty(n)
        active = np.empty(p, dtype=np.int64)
        tp = np.empty(cap, dtype=np.int64)
        ta = np.empty(cap, dtype=np.int64)
        tg = np.empty(cap)
        tr = np.empty(cap)
        history = []
        cb = None
        user_cb = config.on_checkpoint
        if config.track_active or user_cb is not None:
            def _hook(ptr, cnt, _user):
                a = np.ctypeslib.as_array(ptr, shape=(cnt,)).copy() if cnt else np.empty(0, np.int64)
                if config.track_active:
                    history.append(a.copy())
                if user_cb is not None:
                    user_cb(a)
            cb = _lib.CKPT_CB(_hook)
        cfg = _lib.SolveConfig(float(config.epsilon), int(config.max_passes), int(config.screen_every),
                               _GPU_RULES[config.rule], int(bool(config.certify)),
                               cb if cb is not None else _lib.CKPT_CB(), None)
        res = _lib.SolveResult()
        res.beta, res.residual, res.theta, res.active = (_lib.f64p(beta), _lib.f64p(rho),
                                                         _lib.f64p(theta), _lib.i64p(active))
        res.trace_passes, res.trace_active = _lib.i64p(tp), _lib.i64p(ta)
        res.trace_gap, res.trace_radius, res.trace_cap = _lib.f64p(tg), _lib.f64p(tr), cap
        a0 = None
        n0 = 0
        if active0_mode == 1:
            a0 = np.ascontiguousarray(active0, dtype=np.int64)
            n0 = a0.size
        _lib.check(self._lib.gs_solver_solve(self._h, float(lam), ctypes.byref(cfg), _lib.i64p(a0), n0,
                                             int(active0_mode), ctypes.byref(res)))
        nt = res.n_trace
        trace = [(int(tp[i]), int(ta[i]), float(tg[i]), float(tr[i])) for i in range(nt)]
        dual_point = DualPoint(theta=theta, feasibility_margin=float(res.margin),
                               interpolating=bool(res.interpolating))
        cert = GapCertificate(primal=float(res.primal), dual=float(res.dual), gap=float(res.gap))
        state = SolverState(beta=beta, residual=rho, active=active[: res.n_active].copy(),
                            theta=dual_point, cert=cert, passes_done=int(res.passes_done),
                            converged=bool(res.converged), screen_trace=trace,
                            active_history=history)
        state.stats = dict(cd_visits=int(res.cd_visits), cd_uncertified=int(res.cd_uncertified),
                           cd_nonzero=int(res.cd_nonzero), checkpoints=int(res.checkpoints),
                           device_ms=float(res.device_ms), screen_ms=float(res.screen_ms),
                           ckpt_ms=float(res.ckpt_ms), refresh_ms=float(res.refresh_ms),
                           cd_ms=float(res.cd_ms), n_screen=int(res.n_screen),
                           n_refresh=int(res.n_refresh), launches=int(res.launches),
                           cd_candidates=int(res.cd_candidates), cd_skipped=int(res.cd_skipped),
                           cd_requeues=int(res.cd_requeues))
        return beta, cert, state


def _solver_for(prob: LassoProblem) -> DeviceSolver:
    s = getattr(prob, "_device_solver", None)
    if s is None:
        s = DeviceSolver(prob.X, prob.y)
        prob._device_solver = s
    return s


def solve(prob: LassoProblem, config: SolverConfig, warm_beta: np.ndarray | None = None,
          active0: np.ndarray | None = None):
    """Solve one Lasso problem to duality gap <= config.epsilon (solver.py:149-246).

    Returns (beta, GapCertificate, SolverState); ``state.converged`` is
    False when the pass budget ran out."""
    if config.rule not in _GPU_RULES:
        raise NotImplementedError(
            f"rule {config.rule.value!r} is not on the B200 path in this build "
            f"(supported: {', '.join(r.value for r in _GPU_RULES)})")
    if prob.lam > prob.lambda_max * (1 + 1e-12):
        raise ValueError(f"lambda={prob.lam} exceeds lambda_max={prob.lambda_max}")
    if active0 is not None:
        a0 = np.asarray(active0, dtype=np.int64).ravel()
        if a0.size > 1 and not np.all(a0[1:] > a0[:-1]):
            # the reference visits active0 in the given order, duplicates
            # included (solver.py:171-174); the device CD visits an ascending,
            # duplicate-free active set, so any other order is refused loudly
            raise NotImplementedError("active0 must be strictly ascending on the B200 path "
                                      "(as a screen's active_set is)")
    dev = _solver_for(prob)
    dev.set_beta(warm_beta)
    if active0 is None:
        return dev.solve(prob.lam, config)
    return dev.solve(prob.lam, config, active0=active0, active0_mode=1)


class PathTimer:
    """Device-side timing for benchmarks: CUDA events on the solver's stream,
    the standalone full-p screening pass, and the end-to-end path through the
    public API from pinned host buffers."""

    def __init__(self, dev: DeviceSolver):
        self.dev = dev

    def start(self) -> None:
        _lib.check(self.dev._lib.gs_solver_timer(self.dev._h, 0, None))

    def stop_ms(self) -> float:
        ms = ctypes.c_double()
        _lib.check(self.dev._lib.gs_solver_timer(self.dev._h, 1, ctypes.byref(ms)))
        return ms.value

    @staticmethod
    def screen_pass_ms(X, center: np.ndarray, radius: float, reps: int = 10) -> float:
        c = np.ascontiguousarray(center, dtype=np.float64)
        ms = ctypes.c_double()
        cnt = ctypes.c_int64()
        _lib.check(X._lib.gs_screen_timed(X.handle, _lib.f64p(c), float(radius), int(reps),
                                          ctypes.byref(ms), ctypes.byref(cnt), None))
        return ms.value

    @staticmethod
    def screen_pass_active(X, center: np.ndarray, radius: float) -> np.ndarray:
        """Survivors of the fused in-kernel screening pass (the persistent
        kernel's sequential screen, regions.py:129-139 semantics), ascending."""
        c = np.ascontiguousarray(center, dtype=np.float64)
        ms = ctypes.c_double()
        cnt = ctypes.c_int64()
        out = np.empty(X.n_cols, dtype=np.int32)
        _lib.check(X._lib.gs_screen_timed(X.handle, _lib.f64p(c), float(radius), 1,
                                          ctypes.byref(ms), ctypes.byref(cnt), _lib.i32p(out)))
        return out[: cnt.value].astype(np.int64)

    @staticmethod
    def e2e_path_ms(case, grid, config, reps: int = 1):
        """Wall time of DesignMatrix(host X) + DeviceSolver(host y) + run_path
        (coefficients back to host), X and y in pinned host memory."""
        import time as _time
        from .design_matrix import DesignMatrix
        from .path import run_path
        Xh = case.X
        px = _lib.PinnedArray(Xh.shape[::-1], dtype=Xh.dtype)     # (p, n) C-order == (n, p) F-order
        px.array[...] = Xh.T
        py = _lib.PinnedArray(case.y.shape)
        py.array[...] = case.y
        Xf = px.array.T
        best = None
        for _ in range(reps):
            t0 = _time.perf_counter()
            X = DesignMatrix(Xf)
            dev = DeviceSolver(X, py.array)
            res = run_path(X, py.array, grid, config, solver=dev)
            dt = (_time.perf_counter() - t0) * 1e3
            best = dt if best is None else min(best, dt)
            del dev, X
        h2d = Xh.nbytes + case.y.nbytes
        d2h = res.betas.nbytes + sum(s.residual.nbytes + s.theta.theta.nbytes + s.active.nbytes
                                     for s in res.states)
        return best, int(h2d), int(d2h)


class BatchPathSolver:
    """Independent Lasso paths on row-resampled copies of one design
    (BASELINE configs[4], stability selection).  Problem b uses rows
    ``rows[b]`` (with repetition) of ``X0`` and of ``y0``.  All problems run
    concurrently, one CTA each, with the whole warm-started lambda path on the
    device (no per-lambda synchronisation between problems)."""

    def __init__(self, X0, y0: np.ndarray, rows: np.ndarray):
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        if rows.ndim != 2:
            raise ValueError("rows must be (B, n)")
        self.B, self.n = rows.shape
        self.p = X0.n_cols
        self._lib = X0._lib
        y0 = np.ascontiguousarray(y0, dtype=np.float64)
        h = ctypes.c_void_p()
        _lib.check(self._lib.gs_batch_create(X0.handle, _lib.f64p(y0), _lib.i32p(rows), self.B, self.n,
                                             ctypes.byref(h)))
        self._h = h
        lm = np.empty(self.B)
        _lib.check(self._lib.gs_batch_lambda_max(h, _lib.f64p(lm)))
        self.lambda_max = lm

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.gs_batch_free(h)
            self._h = None

    def run_paths(self, grids: np.ndarray, config: SolverConfig, want_betas: bool = False,
                  epsilons: np.ndarray | None = None):
        """grids: (B, T) non-increasing per row.  ``epsilons``: per-problem gap
        tolerances (B,), overriding ``config.epsilon`` (the reference's solve
        takes epsilon per problem, solver.py:37,226; configs[4] uses
        1e-8 * ||y_b||^2).  Returns a dict of (B, T) arrays: passes, gaps,
        converged, n_active (+ betas (B, T, p)) and the device time in ms."""
        if config.rule not in _BATCH_RULES:
            raise NotImplementedError(f"rule {config.rule.value!r} is not on the batched B200 path in this build")
        grids = np.ascontiguousarray(grids, dtype=np.float64)
        B, T = grids.shape
        if B != self.B:
            raise ValueError("grids must have one row per problem")
        if np.any(np.diff(grids, axis=1) > 0):
            raise ValueError("grid must be non-increasing")
        if epsilons is not None:
            epsilons = np.ascontiguousarray(epsilons, dtype=np.float64)
            if epsilons.shape != (B,):
                raise ValueError("epsilons must have one entry per problem")
            if not np.all(epsilons > 0):
                raise ValueError("epsilon must be positive")
        cfg = _lib.SolveConfig(float(config.epsilon), int(config.max_passes), int(config.screen_every),
                               _GPU_RULES[config.rule], int(bool(config.certify)), _lib.CKPT_CB(), None)
        passes = np.empty((B, T), dtype=np.int64)
        gaps = np.empty((B, T))
        conv = np.empty((B, T), dtype=np.int32)
        nact = np.empty((B, T), dtype=np.int64)
        betas = np.empty((B, T, self.p)) if want_betas else None
        ms = ctypes.c_double()
        _lib.check(self._lib.gs_batch_run_paths(self._h, _lib.f64p(grids), T, ctypes.byref(cfg),
                                                _lib.f64p(epsilons), _lib.f64p(betas), _lib.i64p(passes), _lib.f64p(gaps),
                                                _lib.i32p(conv), _lib.i64p(nact), ctypes.byref(ms)))
        out = dict(passes=passes, gaps=gaps, converged=conv.astype(bool), n_active=nact, device_ms=ms.value)
        if want_betas:
            out["betas"] = betas
        return out
