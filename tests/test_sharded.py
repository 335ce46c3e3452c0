"""Column-sharded path (paper_1505_03410_b200/sharded.py).

CPU (gloo, world size 2): the sharded driver -- arg-max lambda_max across
shards, column-parallel sequential screen, survivors gathered to rank 0 --
run with the oracle as its compute backend reproduces the single-process
oracle path (tests/parity.py criteria: the sub-solve's BLAS products run over
the gathered columns, so coefficients/gaps agree to round-off).

GPU (-m gpu, gloo on one device): the same driver with the product backend
(sm_100a kernels) against the single-process oracle path.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleBackend:
    """Test-only backend: the CPU oracle behind sharded.py's interface."""

    def __init__(self, X_block, y):
        from oracle import gapsafe_oracle as O
        self.O = O
        self.Xh = X_block
        self.X = O.DesignMatrix(X_block)
        self.y = np.ascontiguousarray(y, dtype=np.float64)

    @property
    def n_cols(self):
        return self.X.n_cols

    def max_abs_correlation(self, v):
        return self.X.max_abs_correlation(v)

    def screen(self, center, radius, tol=1e-9):
        O = self.O
        return O.screen(O.Sphere(center=center, radius=float(radius)), self.X, tol).active_set

    def columns(self, idx):
        # (k, n) tensor on the communication device, like DeviceBackend.columns
        return torch.from_numpy(np.ascontiguousarray(self.Xh[:, idx].T))

    def solve_sub(self, XA, lam, lambda_max, warm_beta, config):
        O = self.O
        XA = np.asfortranarray(XA.numpy().T)
        prob = O.LassoProblem(O.DesignMatrix(XA), self.y, lam, lambda_max=(lambda_max, 0))
        ocfg = O.SolverConfig(epsilon=config.epsilon, max_passes=config.max_passes,
                              screen_every=config.screen_every, rule=config.rule.value)
        return O.solve(prob, ocfg, warm_beta=warm_beta, active0=np.arange(XA.shape[1], dtype=np.int64))


def _case():
    from paper_1505_03410_b200 import synth
    c = synth.cfg0(p=1300)
    from oracle import gapsafe_oracle as O
    lmax, _ = O.DesignMatrix(c.X).max_abs_correlation(c.y)
    grid = O.lambda_grid(lmax, 12, 2.5)
    return c, grid


def _worker(rank, world, port, q, device):
    import torch.distributed as dist
    from paper_1505_03410_b200 import dist as D
    from paper_1505_03410_b200 import sharded
    from paper_1505_03410_b200.solver import SolverConfig
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, grid = _case()
        p = c.X.shape[1]
        lo, hi = D.shard_range(p, rank, world)
        block = np.asfortranarray(c.X[:, lo:hi])
        be = sharded.DeviceBackend(block, c.y) if device else OracleBackend(block, c.y)
        res = sharded.run_path_sharded(be, c.y, grid, SolverConfig(epsilon=c.epsilon, max_passes=100_000), p, lo)
        if rank == 0:
            q.put(("ok", [(s.beta, s.passes_done, s.converged, s.active, s.screen_trace, s.cert.gap)
                          for s in res.states]))
        else:
            q.put(("ok", None))
    except Exception as e:  # surface worker failures in the test
        import traceback
        q.put(("err", traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _run(device):
    from oracle import gapsafe_oracle as O
    from parity import compare_paths
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, device)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    errs = [o[1] for o in outs if o[0] == "err"]
    assert not errs, errs[0]
    got = next(o[1] for o in outs if o[1] is not None)
    c, grid = _case()
    ref = O.run_path(O.DesignMatrix(c.X), c.y, grid, O.SolverConfig(epsilon=c.epsilon, max_passes=100_000))

    class _S:
        pass

    class _R:
        pass

    ra = _R()
    ra.states = []
    for beta, passes, conv, act, trace, gap in got:
        s = _S()
        s.beta, s.passes_done, s.converged, s.active, s.screen_trace = beta, passes, conv, act, trace
        s.cert = _S()
        s.cert.gap = gap
        ra.states.append(s)
    ra.converged = np.array([s.converged for s in ra.states])
    compare_paths(ra, ref, float(c.y @ c.y))


def test_sharded_path_gloo_oracle_backend():
    _run(device=False)


@pytest.mark.gpu
def test_sharded_path_device_backend():
    _run(device=True)


def _batch_worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_1505_03410_b200 as gs
    from paper_1505_03410_b200 import sharded, synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X0, y0, _ = synth.cfg4_shared(p=3000)
        B = 6
        rows = np.stack([synth.cfg4_rows(b) for b in range(B)]).astype(np.int32)
        D0 = gs.DesignMatrix(X0)
        lm = gs.BatchPathSolver(D0, y0, rows).lambda_max
        grids = np.stack([gs.lambda_grid(lm[b], 8, 2.0) for b in range(B)])
        cfg = gs.SolverConfig(epsilon=1e-8 * float(y0 @ y0) / 2, max_passes=100_000)
        res, _ = sharded.run_batch_sharded(D0, y0, rows, grids, cfg)
        if rank == 0:
            single = gs.BatchPathSolver(D0, y0, rows).run_paths(grids, cfg)
            q.put(("ok", (res, single)))
        else:
            q.put(("ok", None))
    except Exception:
        import traceback
        q.put(("err", traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_batch_problem_sharding_matches_single_process():
    """cfg4 problem sharding: two ranks, three problems each, identical per-problem
    epochs / gaps / active-set sizes to one process running all six."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    errs = [o[1] for o in outs if o[0] == "err"]
    assert not errs, errs[0]
    res, single = next(o[1] for o in outs if o[1] is not None)
    assert np.array_equal(res["passes"], single["passes"])
    assert np.array_equal(res["n_active"], single["n_active"])
    assert np.array_equal(res["converged"], single["converged"])
    assert np.array_equal(res["gaps"], single["gaps"])
