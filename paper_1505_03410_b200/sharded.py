"""Column-sharded Lasso path over one process per GPU.

Rank g owns the contiguous column block [lo_g, hi_g) of X (``dist.shard_range``)
in its own HBM.  Per grid point (path.py:52-105):

  * lambda_max = |X^T y|_inf and j* (problem.py:41-54): each rank runs the
    fused screening GEMV over its block; the global arg-max (smallest index on
    ties, design_matrix.py:160-174) is an all-gather of 16 bytes -- once per
    path;
  * lambda >= lambda_max (solver.py:129-146): theta = y / lambda, r = 0, the
    sphere test runs column-parallel on every rank;
  * the sequential gap-sphere screen (path.py:82-91): rank 0 holds the
    previous (beta, theta, rho) and computes G_t and r_t (problem.py:57-86,
    regions.py:213-218); theta_prev and r_t are broadcast (n*8 + 8 bytes);
    every rank runs the fused full-block screen (the HBM-bound pass, 1/k of
    the design per GPU) and the survivors' indices are gathered;
  * solve (solver.py:149-246): the survivors' columns X_A are gathered to
    rank 0 ("gather X_A" alternative of §8(e); |A| n s bytes over NVLink) and
    solved there with the path's lambda_max -- every operation of solve()
    except the lambda_max shortcut is restricted to A, so this is solve(prob,
    active0=A) on the full design.

Backends: ``DeviceBackend`` (the product: sm_100a kernels through the C ABI)
and, in the tests only, an oracle backend with the same interface.
Collectives go through torch.distributed (NCCL on the GPU box, gloo in the
CPU tests); results are assembled on rank 0.
"""

from __future__ import annotations

import time

import numpy as np

from . import dist as D
from .path import PathResult
from .problem import DualPoint, GapCertificate, LassoProblem, InfeasibleDualError
from .regions import NumericalInconsistencyError, SCREEN_SAFETY, Sphere, screen
from .solver import Rule, SolverConfig, SolverState


class DeviceBackend:
    """Per-rank compute on the B200: the local column block lives in HBM.

    The survivors' columns never visit the host: ``columns`` gathers them into
    a CUDA tensor (the NCCL send buffer) with a device kernel, and
    ``solve_sub`` builds rank 0's sub-design from the received tensor with a
    device-to-device copy (``DesignMatrix.from_device``)."""

    def __init__(self, X_block, y):
        from .design_matrix import DesignMatrix
        self.X = X_block if isinstance(X_block, DesignMatrix) else DesignMatrix(X_block)
        if self.X.is_sparse:
            raise NotImplementedError("the column-sharded path gathers dense columns")
        self.y = np.ascontiguousarray(y, dtype=np.float64)

    @property
    def n_cols(self) -> int:
        return self.X.n_cols

    def max_abs_correlation(self, v):
        return self.X.max_abs_correlation(np.ascontiguousarray(v, dtype=np.float64))

    def screen(self, center, radius, tol=SCREEN_SAFETY) -> np.ndarray:
        return screen(Sphere(center=np.ascontiguousarray(center, dtype=np.float64), radius=float(radius)),
                      self.X, tol).active_set

    def columns(self, idx):
        """(k, n) tensor of the local columns ``idx`` on this rank's GPU."""
        import torch
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        n = self.X.n_base
        tdt = torch.float32 if self.X.dtype == np.float32 else torch.float64
        buf = torch.empty((max(1, idx.size), n), dtype=tdt, device=torch.device("cuda", torch.cuda.current_device()))
        if idx.size:
            self.X.gather_columns_to_device(idx, buf.data_ptr(), n)
        return buf[: idx.size]

    def solve_sub(self, XA, lam, lambda_max, warm_beta, config):
        """solve(prob, config, warm_beta, active0=all) on the gathered design
        (a (k, n) CUDA tensor) with the full path's lambda_max (no shortcut
        below it)."""
        import torch
        from .design_matrix import DesignMatrix
        from .solver import DeviceSolver
        k, n = int(XA.shape[0]), int(XA.shape[1])
        torch.cuda.synchronize()              # the gather (NCCL stream) has written XA
        D_A = DesignMatrix.from_device(XA.data_ptr(), n, k, n, np.float32 if XA.dtype == torch.float32 else np.float64)
        dev = DeviceSolver(D_A, self.y)
        dev.set_lambda_max(lambda_max)
        dev.set_beta(warm_beta)
        return dev.solve(lam, config, active0=np.arange(k, dtype=np.int64), active0_mode=1)


def _bcast_array(a, src: int = 0):
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(D._device())
    dist.broadcast(t, src)
    return t.cpu().numpy()


def _gather_int(x: np.ndarray, world: int) -> list[np.ndarray]:
    """All-gather of variable-length int64 arrays (counts first, then padded)."""
    import torch
    import torch.distributed as dist
    dev = D._device()
    cnt = torch.tensor([x.size], dtype=torch.int64, device=dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    cnts = [int(c.item()) for c in cnts]
    mx = max(1, max(cnts))
    buf = torch.zeros(mx, dtype=torch.int64, device=dev)
    buf[: x.size] = torch.as_tensor(x, dtype=torch.int64)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    return [o[:c].cpu().numpy() for o, c in zip(outs, cnts)]


def _gather_columns(cols, n: int, world: int, rank: int):
    """Gather every rank's (k_g, n) column tensor to rank 0, in rank order.
    The tensors stay on the communication device (GPU memory under NCCL: the
    transfer is device to device over NVLink); rank 0 gets the (sum k_g, n)
    tensor, the others None."""
    import torch
    import torch.distributed as dist
    k = int(cols.shape[0])
    ks = _gather_int(np.array([k], dtype=np.int64), world)
    ks = [int(a[0]) for a in ks]
    mx = max(1, max(ks))
    # under NCCL the buffers are the GPU tensors themselves; only the gloo
    # fallback of the 1-GPU test box (ranks sharing a device) stages on the host
    comm = D._device()
    buf = torch.zeros((mx, n), dtype=cols.dtype, device=comm)
    if k:
        buf[:k] = cols
    outs = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, outs, dst=0)
    if rank != 0:
        return None
    return torch.cat([o[:kk] for o, kk in zip(outs, ks)], dim=0).to(cols.device)


_ST_OK, _ST_INFEASIBLE, _ST_NUMERICAL, _ST_OTHER = 0, 1, 2, 3


def _sync_status(exc: BaseException | None, src: int = 0) -> None:
    """Rank ``src`` reports the exception it caught (or None); every rank
    learns the status word and raises together, so no rank is left blocked in
    the next collective when the reference's synchronous errors
    (InfeasibleDualError / NumericalInconsistencyError, solver.py:219-221)
    fire on rank 0."""
    import torch.distributed as dist
    code = _ST_OK
    if exc is not None:
        code = (_ST_INFEASIBLE if isinstance(exc, InfeasibleDualError)
                else _ST_NUMERICAL if isinstance(exc, NumericalInconsistencyError) else _ST_OTHER)
    code = int(_bcast_array([float(code)], src)[0])
    if code == _ST_OK:
        return
    if exc is not None and dist.get_rank() == src:
        raise exc
    if code == _ST_INFEASIBLE:
        raise InfeasibleDualError(f"dual point infeasible on rank {src}")
    if code == _ST_NUMERICAL:
        raise NumericalInconsistencyError(f"numerical inconsistency reported by rank {src}")
    raise RuntimeError(f"rank {src} failed; see its traceback")


def run_path_sharded(backend, y: np.ndarray, grid: np.ndarray, config: SolverConfig, p_total: int,
                     col_lo: int) -> PathResult | None:
    """Warm-started Gap Safe path over a column-sharded design (see module
    docstring).  Every rank calls it with its own backend/column offset;
    rank 0 returns the PathResult (coefficients over all ``p_total``
    columns), the other ranks return None."""
    import torch.distributed as dist
    if config.rule not in (Rule.NONE, Rule.GAP_SPHERE):
        raise NotImplementedError("the sharded path runs the none / gap_sphere rules (north_star)")
    rank, world = dist.get_rank(), dist.get_world_size()
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = y.size
    grid = np.asarray(grid, dtype=np.float64)
    if grid.size == 0:
        raise ValueError("empty lambda grid")
    if np.any(np.diff(grid) > 0):
        raise ValueError("grid must be non-increasing")
    v, j = backend.max_abs_correlation(y)
    lmax, jstar = D.argmax_over_ranks(float(v), col_lo + int(j))
    y_norm_sq = float(np.dot(y, y))
    T = grid.size
    betas = np.zeros((T, p_total)) if rank == 0 else None
    certs, traces, timings, states = [], [], [], []
    conv = np.zeros(T, dtype=bool)
    prev = None          # rank 0: (beta dense, theta DualPoint, rho)
    for t, lam in enumerate(grid):
        t0 = time.perf_counter()
        if lam <= 0:
            raise ValueError("lambda must be positive")
        if lam > lmax * (1 + 1e-12):
            raise ValueError(f"lambda={lam} exceeds lambda_max={lmax}")
        if lam >= lmax * (1 - 1e-14):
            # _solve_at_lambda_max (solver.py:129-146): the sphere test at r = 0
            theta = y / lam
            if config.rule is Rule.NONE:
                loc = np.arange(backend.n_cols, dtype=np.int64)[_nonzero_norms(backend)]
            else:
                loc = backend.screen(theta, 0.0)
            act = np.concatenate(_gather_int(col_lo + loc.astype(np.int64), world))
            if rank == 0:
                beta = np.zeros(p_total)
                dp = DualPoint(theta=theta, feasibility_margin=0.0)
                cert = GapCertificate(primal=0.5 * y_norm_sq, dual=0.5 * y_norm_sq, gap=0.0)
                state = SolverState(beta=beta, residual=y.copy(), active=act, theta=dp, cert=cert,
                                    passes_done=0, converged=True, screen_trace=[(0, int(act.size), 0.0, 0.0)])
                prev = (beta, dp, y.copy())
        else:
            seq = (t > 0 and config.rule is Rule.GAP_SPHERE)
            if seq:
                interp = _bcast_array([1.0 if (rank == 0 and prev[1].interpolating) else 0.0])[0] > 0
                seq = not interp
            if seq:
                # G_t = P_t(beta_prev) - D_t(theta_prev) with rho_prev (problem.py:57-86)
                hdr = np.zeros(n + 1)
                err = None
                if rank == 0:
                    try:
                        beta_p, th_p, rho_p = prev
                        if th_p.feasibility_margin < -1e-9:
                            raise InfeasibleDualError(f"dual point infeasible: margin={th_p.feasibility_margin}")
                        primal = 0.5 * float(np.dot(rho_p, rho_p)) + lam * float(np.sum(np.abs(beta_p)))
                        diff = th_p.theta - y / lam
                        dual = 0.5 * y_norm_sq - 0.5 * lam ** 2 * float(np.dot(diff, diff))
                        gap = primal - dual
                        if gap < -1e-10:
                            raise NumericalInconsistencyError(f"negative duality gap beyond tolerance: {gap}")
                        hdr[:n] = th_p.theta
                        hdr[n] = float(np.sqrt(2.0 * max(gap, 0.0)) / lam)
                    except Exception as e:       # reported to every rank below
                        err = e
                _sync_status(err)
                hdr = _bcast_array(hdr)
                loc = backend.screen(hdr[:n], hdr[n])
            else:
                loc = np.arange(backend.n_cols, dtype=np.int64)[_nonzero_norms(backend)]
            glob = _gather_int(col_lo + loc.astype(np.int64), world)
            act = np.concatenate(glob)
            XA = _gather_columns(backend.columns(loc), n, world, rank)
            err = None
            if rank == 0:
                try:
                    beta_full = prev[0] if prev is not None else np.zeros(p_total)
                    bA, cert, st = backend.solve_sub(XA, float(lam), lmax, beta_full[act], config)
                except Exception as e:
                    err = e
            _sync_status(err)
            if rank == 0:
                beta = np.zeros(p_total)
                beta[act] = bA
                state = SolverState(beta=beta, residual=st.residual, active=act[st.active], theta=st.theta,
                                    cert=cert, passes_done=st.passes_done, converged=st.converged,
                                    screen_trace=st.screen_trace, active_history=st.active_history)
                state.stats = getattr(st, "stats", {})
                prev = (beta, st.theta, st.residual)
        timings.append(time.perf_counter() - t0)
        if rank == 0:
            betas[t] = state.beta
            certs.append(state.cert)
            traces.append(state.screen_trace)
            states.append(state)
            conv[t] = state.converged
    if rank != 0:
        return None
    return PathResult(lambdas=grid, betas=betas, certs=certs, traces=traces, timings=timings,
                      converged=conv, states=states)


def _nonzero_norms(backend) -> np.ndarray:
    norms = backend.X.col_norms if hasattr(backend, "X") else backend.col_norms
    return np.asarray(norms) > 0


def run_batch_sharded(X0, y0: np.ndarray, rows: np.ndarray, grids: np.ndarray, config: SolverConfig,
                      epsilons: np.ndarray | None = None):
    """Independent problems sharded by problem index:
    rank g runs problems ``shard_range(B, g, world)`` with one CTA each on its
    own GPU (``BatchPathSolver``); X0 and y0 are replicated.  No collective on
    the data path -- rank 0 gathers the per-problem (passes, gaps, converged,
    n_active) at the end.  Returns the full (B, T) arrays on rank 0, None
    elsewhere, plus the local device time (ms) on every rank."""
    import torch
    import torch.distributed as dist
    from .solver import BatchPathSolver
    rank, world = dist.get_rank(), dist.get_world_size()
    B = rows.shape[0]
    lo, hi = D.shard_range(B, rank, world)
    T = grids.shape[1]
    out = None
    if hi > lo:
        bs = BatchPathSolver(X0, y0, rows[lo:hi])
        out = bs.run_paths(grids[lo:hi], config, epsilons=None if epsilons is None else epsilons[lo:hi])
    dev = D._device()
    mx = max(D.shard_range(B, r, world)[1] - D.shard_range(B, r, world)[0] for r in range(world))
    pack = torch.zeros((mx, T, 4), dtype=torch.float64, device=dev)
    if out is not None:
        loc = np.stack([out["passes"], out["gaps"], out["converged"], out["n_active"]], axis=-1).astype(np.float64)
        pack[: hi - lo] = torch.as_tensor(loc)
    parts = [torch.zeros_like(pack) for _ in range(world)] if rank == 0 else None
    dist.gather(pack, parts, dst=0)
    ms = out["device_ms"] if out is not None else 0.0
    if rank != 0:
        return None, ms
    full = np.concatenate([parts[r][: D.shard_range(B, r, world)[1] - D.shard_range(B, r, world)[0]].cpu().numpy()
                           for r in range(world)], axis=0)
    res = dict(passes=full[..., 0].astype(np.int64), gaps=full[..., 1], converged=full[..., 2] > 0,
               n_active=full[..., 3].astype(np.int64))
    return res, ms
