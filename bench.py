"""Benchmark: Lasso-path wall time to gap 1e-8 (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg0|cfg1|cfg2|cfg3|cfg4] [--impl ours|reference]

A "step" is one full warm-started Gap Safe Lasso path over the config's
lambda grid.  ``value`` is the path wall time measured on
the device with CUDA events bracketing the path on the solver's stream
(inputs resident in HBM); ``e2e`` is the same path through the public API
from pinned host buffers (design + response H2D, coefficients D2H inside the
timed region).  At N > 1 every rank runs an independent replica of the path
(cfg1 does not shard: "replicas only"); the reported time is the
max over ranks.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port of /root/reference/pkg/src/gapsafe, bit-identical to it, see
tests/test_oracle_golden.py) on the same workload: complete paths, as many as
fit its time budget (the line reports how many ran).

After the timed steps rank 0 checks the benchmarked path against the oracle
on its first lambdas (``parity`` block: epochs, per-checkpoint active sets,
supports, beta, gaps) and exits non-zero on a mismatch.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Lasso-path wall time to gap 1e-8 (s); screening-pass HBM GB/s vs peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 5 + k and r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _init_ranks(ws, local):
    """One process per GPU (NCCL).  When the box has fewer GPUs than ranks (the
    1-GPU test box), ranks share devices and the host collectives run over
    gloo -- no kernel of one rank ever waits on another rank."""
    import torch
    import torch.distributed as dist
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl" if ndev >= ws else "gloo")
    return dev


def _make_case(name, p=None):
    from paper_1505_03410_b200 import synth
    return synth.by_name(name, **({} if p is None else {"p": int(p)}))


def _grid(lmax, case):
    from paper_1505_03410_b200 import lambda_grid
    return lambda_grid(lmax, case.n_lambdas, case.delta)


def _roofline_traffic(config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the screening
    kernel, from the NEWEST committed ``ncu --set full`` capture of this config
    (profiles/r*/ncu_screen_full_<config>*.md, by round then file time)."""
    import glob
    import re
    cands = glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_screen_full_{config}*.md"))
    cands.sort(key=lambda p: (os.path.basename(os.path.dirname(p)), os.path.getmtime(p)), reverse=True)
    for path in cands:
        try:
            txt = open(path).read()
        except OSError:
            continue
        vals = {}
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            m = re.search(re.escape(key) + r" \| ([0-9.]+) (\w+)", txt)
            if m:
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m.group(2), None)
                if mult:
                    vals[key] = float(m.group(1)) * mult
        if len(vals) == 2:
            return sum(vals.values()), os.path.relpath(path, ROOT)
    return None, None


def _parity_mod():
    import importlib.util
    spec = importlib.util.spec_from_file_location("_bench_parity", os.path.join(ROOT, "tests", "parity.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _cpu_sample(case, grid, budget_s, track=False):
    """Oracle (reference algorithm, CPU) on the first lambdas of the same path,
    stopping after the point at which the budget is exceeded (budget None:
    the whole path)."""
    from oracle import gapsafe_oracle as O
    X = O.DesignMatrix(case.X)
    t0 = time.perf_counter()
    res = O.run_path(X, case.y, grid, O.SolverConfig(epsilon=case.epsilon, max_passes=100_000,
                                                     track_active=track),
                     cache_lambda_max=True, time_budget_s=budget_s)
    wall = time.perf_counter() - t0
    return res, wall


def _workload_config(args, case, grid):
    """The ``config`` object, identical in both arms."""
    n, p = case.X.shape
    es = case.X.dtype.itemsize
    return {"workload": args.config, "n": int(n), "p": int(p), "lambdas": int(grid.size), "tol": case.tol,
            "screen_every": 10, "rule": "gap_sphere",
            "l2": f"design {n * p * es / 1e6:.0f} MB > 126 MB L2: streamed inputs, no flush needed"}


def run_reference(args):
    """The reference algorithm's CPU implementation (the oracle port, pinned
    bit-for-bit to the reference's golden paths) on the SAME workload: every
    timed step is one complete path over all the grid's lambdas.  Steps are
    run while the time budget allows (at least one), and the line reports the
    number actually run; the warm-up steps are the path's first lambdas (BLAS
    threads and the C kernels warm), stated in ``warmup_note``."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    case = _make_case(args.config, args.p)
    from oracle import gapsafe_oracle as O
    O.build_kernels()
    Xo = O.DesignMatrix(case.X)
    lmax, _ = Xo.max_abs_correlation(case.y)
    grid = O.lambda_grid(lmax, case.n_lambdas, case.delta)
    cores = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        O.run_path(Xo, case.y, grid, O.SolverConfig(epsilon=case.epsilon, max_passes=100_000),
                   cache_lambda_max=True, max_points=3)
    times, t_all = [], time.perf_counter()
    while True:
        res, _ = _cpu_sample(case, grid, None)
        times.append(sum(res.timings))
        if len(times) >= args.steps:
            break
        spent = time.perf_counter() - t_all
        if spent + max(times) > args.ref_budget:
            break
    value = statistics.mean(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": ws,
            "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup,
            "warmup_note": "each warm-up step is the first 3 lambdas of the same path",
            "ms_per_step": value * 1e3, "step_s": times,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, SURVEY.md §8(d))",
            "config": _workload_config(args, case, grid),
            "cpu_baseline": {"value": value, "unit": "s", "cores": cores, "kind": "port",
                             "sample": f"complete {args.config} path ({grid.size} lambdas, run_path timing scope "
                                       f"path.py:78,94); OpenBLAS on {cores} threads, CD kernels single-threaded "
                                       f"as in the reference",
                             "epochs": int(sum(s.passes_done for s in res.states))},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _gpu_parity(case, grid, cfg_cls, X, dev, k_budget_s, ynsq):
    """Parity of the benchmarked path against the oracle on its first
    lambdas: the oracle runs the path with per-checkpoint active sets tracked
    until ``k_budget_s`` is spent (k lambdas); the device re-runs the same k
    lambdas with tracking.  Epochs, per-checkpoint active sets (element by
    element), supports, beta (1e-8 rel) and gaps (D7 floor) are compared."""
    import paper_1505_03410_b200 as gs
    ref, wall = _cpu_sample(case, grid, k_budget_s, track=True)
    k = len(ref.states)
    cfg = gs.SolverConfig(epsilon=case.epsilon, max_passes=100_000, track_active=True)
    mine = gs.run_path(X, case.y, grid[:k], cfg, solver=dev)
    rep = _parity_mod().path_report(mine, ref, ynsq)
    rep["oracle_s"] = sum(ref.timings)
    rep["gpu_s"] = sum(mine.timings)
    return rep, ref


def run_ours(args):
    ws, rank, local = _dist()
    import paper_1505_03410_b200 as gs
    from paper_1505_03410_b200 import _lib
    if ws > 1:
        local = _init_ranks(ws, local)
    _lib.init_device(local)
    case = _make_case(args.config, args.p)
    n, p = case.X.shape
    X = gs.DesignMatrix(case.X)
    dev = gs.DeviceSolver(X, case.y)
    grid = _grid(dev.lambda_max, case)
    cfg = gs.SolverConfig(epsilon=case.epsilon, max_passes=100_000)
    timer = gs.PathTimer(dev)

    def one_path():
        timer.start()
        res = gs.run_path(X, case.y, grid, cfg, solver=dev)
        return res, timer.stop_ms()

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        one_path()
    barrier()
    l0 = _lib.launch_count()
    ms, results = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            res, t = one_path()
            ms.append(t)
            results.append(res)
    launches = (_lib.launch_count() - l0) / args.steps
    barrier()
    ms_step = statistics.mean(ms)
    if ws > 1:
        from paper_1505_03410_b200.dist import max_over_ranks
        ms_step = max_over_ranks(ms_step)
    res = results[-1]
    # every timed step must produce the same path (determinism)
    same = all(all(a.passes_done == b.passes_done for a, b in zip(r.states, res.states)) for r in results)
    st = [s.stats for s in res.states]
    agg = {k: sum(x[k] for x in st) for k in ("cd_visits", "cd_uncertified", "cd_nonzero", "checkpoints",
                                             "screen_ms", "ckpt_ms", "refresh_ms", "cd_ms", "n_screen",
                                             "n_refresh")}
    epochs = int(sum(s.passes_done for s in res.states))

    # ---- screening-pass roofline: the fused full-p GEMV + sphere test + compaction
    peak, peak_kind = _peaks()
    es = case.X.dtype.itemsize
    if getattr(X, "is_sparse", False):
        nnz = int(case.X.nnz)
        scr_bytes = nnz * (8 + 4) + 8 * (p + 1) + p * (8 + 1) + n * 8
    else:
        scr_bytes = n * p * es + p * (8 + 1) + n * 8       # X, norms in, keep marks out, center
    # average launch duration of back-to-back launches (CUDA events on the
    # launching stream); median over 3 batches of 20 to damp run-to-run noise
    scr_ms = statistics.median(timer.screen_pass_ms(X, res.states[-1].theta.theta, 1e-3, reps=20) for _ in range(3))
    achieved = scr_bytes / (scr_ms * 1e-3) / 1e9
    traffic, traffic_src = _roofline_traffic(args.config)
    inpath_screen = agg["screen_ms"] / max(1, agg["n_screen"])

    # ---- e2e through the public API from pinned host buffers
    e2e_ms, h2d, d2h = timer.e2e_path_ms(case, grid, cfg, reps=1)

    line = {
        "metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md §8(d))",
        "config": _workload_config(args, case, grid),
        "parallelism": "replicas" if ws > 1 else "single",
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "k_screen_full (group_gemv G_MU: full-p screening GEMV + sphere test)",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "bytes_per_launch": scr_bytes, "launch_ms": scr_ms,
                     "in_path_screen_ms": inpath_screen},
        "e2e": {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "path": {"epochs": epochs, "checkpoints": agg["checkpoints"], "converged": int(res.converged.sum()),
                 "steps_identical": bool(same),
                 "cd_visits": agg["cd_visits"], "cd_uncertified": agg["cd_uncertified"],
                 "cd_nonzero": agg["cd_nonzero"], "refreshes": agg["n_refresh"],
                 "phase_ms": {"screen": agg["screen_ms"], "checkpoint": agg["ckpt_ms"],
                              "refresh": agg["refresh_ms"], "cd": agg["cd_ms"]},
                 "cd_updates_per_s": agg["cd_uncertified"] / max(1e-9, agg["cd_ms"] * 1e-3)},
    }
    ok = True
    if rank == 0 and ws == 1 and not args.no_cpu:
        ynsq = float(case.y @ case.y)
        par, ref = _gpu_parity(case, grid, None, X, dev, args.cpu_budget, ynsq)
        line["parity"] = par
        ok = bool(par["ok"])
        k = par["lambdas_compared"]
        gpu_same = sum(res.timings[:k])
        measured = sum(ref.timings)
        line["cpu_baseline"] = {"value": measured, "unit": "s", "cores": len(os.sched_getaffinity(0)),
                                "kind": "port",
                                "sample": (f"first {k} of {grid.size} lambdas of the {args.config} path (oracle, "
                                           f"run_path timing scope path.py:78,94; not scaled); the complete path "
                                           f"is timed by the reference arm (bench.py --impl reference)"),
                                "gpu_same_sample_s": gpu_same,
                                "speedup_same_sample": measured / max(gpu_same, 1e-12)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if not ok:
        print("bench: PARITY FAILURE against the oracle: " + str(line["parity"].get("first_mismatch")),
              file=sys.stderr, flush=True)
        return 3
    return 0


def run_cfg4(args):
    """configs[4]: B bootstrap problems (n = 500 rows drawn with replacement from
    the shared 1000 x p design), each a 50-lambda path to lambda_max / 100 at
    its own tolerance eps_b = 1e-8 ||y_b||^2, sharded by problem index over
    the ranks (sharded.run_batch_sharded: no collective on the data path).  A
    step is the whole batch; the time is the max over ranks of the device time
    of the rank's persistent batch kernel.  Total work is fixed: "strong"."""
    ws, rank, local = _dist()
    import paper_1505_03410_b200 as gs
    from paper_1505_03410_b200 import _lib, sharded, synth
    from paper_1505_03410_b200 import dist as D
    if ws > 1:
        local = _init_ranks(ws, local)
    _lib.init_device(local)
    B, T = int(args.problems), 50
    X0, y0, _ = synth.cfg4_shared(p=args.p or 50_000)
    rows = np.stack([synth.cfg4_rows(b) for b in range(B)]).astype(np.int32)
    D0 = gs.DesignMatrix(X0)
    lo, hi = D.shard_range(B, rank, ws)
    t0 = time.perf_counter()
    bs = gs.BatchPathSolver(D0, y0, rows[lo:hi]) if hi > lo else None
    setup_s = time.perf_counter() - t0
    lmax = bs.lambda_max if bs is not None else np.zeros(0)
    grids = np.stack([gs.lambda_grid(lmax[b - lo], T, 2.0) for b in range(lo, hi)]) if hi > lo else np.zeros((0, T))
    eps = np.array([1e-8 * float(y0[rows[b]] @ y0[rows[b]]) for b in range(lo, hi)])
    cfg = gs.SolverConfig(epsilon=1.0, max_passes=100_000)

    def step():
        if bs is None:
            return None, 0.0
        out = bs.run_paths(grids, cfg, epsilons=eps)
        return out, out["device_ms"]

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup if not args.quick else 0):
        step()
    barrier()
    l0 = _lib.launch_count()
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            out, dms = step()
            wall = (time.perf_counter() - t0) * 1e3
            ms.append((dms, wall))
    launches = (_lib.launch_count() - l0) / args.steps
    barrier()
    ms_step = statistics.mean(m[0] for m in ms)
    e2e_ms = statistics.mean(m[1] for m in ms) + setup_s * 1e3      # + gather / norms / lambda_max of the shard
    if ws > 1:
        ms_step = D.max_over_ranks(ms_step)
        e2e_ms = D.max_over_ranks(e2e_ms)
    n, p = rows.shape[1], X0.shape[1]
    peak, peak_kind = _peaks()
    scr_bytes = X0.shape[0] * p * 8 + p * 9 + X0.shape[0] * 8
    scr_ms = gs.PathTimer.screen_pass_ms(D0, y0 / float(np.max(np.abs(X0.T @ y0))), 1e-3, reps=20)
    line = {"metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, SURVEY.md §8(d))",
            "config": {"workload": "cfg4", "problems": B, "n": int(n), "p": int(p), "lambdas": T, "tol": 1e-8,
                       "eps": "per problem, 1e-8 ||y_b||^2", "screen_every": 10, "rule": "gap_sphere",
                       "l2": f"{hi - lo} resampled designs of {n * p * 8 / 1e6:.0f} MB each > 126 MB L2"},
            "parallelism": f"problems sharded over {ws} rank(s)", "clocks": clk.summary(), "gpu_launches": launches,
            "roofline": {"bound": "hbm", "kernel": "k_screen_full on the shared design", "achieved": scr_bytes / (scr_ms * 1e-3) / 1e9,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": scr_bytes / (scr_ms * 1e-3) / 1e9 / peak, "traffic": None,
                         "bytes_per_launch": scr_bytes, "launch_ms": scr_ms},
            "e2e": {"value": e2e_ms / 1e3, "unit": "s", "h2d_bytes_per_step": int(X0.nbytes + y0.nbytes + rows[lo:hi].nbytes),
                    "d2h_bytes_per_step": int((hi - lo) * T * 28)}}
    if out is not None:
        line["path"] = {"epochs": int(out["passes"].sum()), "converged": int(out["converged"].sum()), "of": int((hi - lo) * T),
                        "rank0_problems": [int(lo), int(hi)]}
    ok = True
    if rank == 0 and not args.no_cpu and out is not None:
        # parity + CPU baseline: the oracle on problem `lo`, first lambdas within the budget
        from oracle import gapsafe_oracle as O
        Xb = np.asfortranarray(X0[rows[lo]])
        yb = y0[rows[lo]]
        ref = O.run_path(O.DesignMatrix(Xb), yb, grids[0], O.SolverConfig(epsilon=float(eps[0]), max_passes=100_000),
                         cache_lambda_max=True, time_budget_s=args.cpu_budget)
        k = len(ref.states)
        same = all(int(out["passes"][0, t]) == ref.states[t].passes_done and
                   int(out["n_active"][0, t]) == ref.states[t].active.size for t in range(k))
        ok = bool(same)
        line["parity"] = {"problem": int(lo), "lambdas_compared": k, "epochs_and_active_sizes_equal": ok, "ok": ok}
        line["cpu_baseline"] = {"value": float(sum(ref.timings)), "unit": "s", "cores": len(os.sched_getaffinity(0)),
                                "kind": "port", "sample": f"first {k} of {T} lambdas of problem {lo} (1 of {B} problems; oracle)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0 if ok else 3


def run_cfg2_sharded(args):
    """configs[2] at N > 1: the design is sharded by contiguous column blocks
    (each rank generates and uploads only its own columns), the full-p
    screening pass runs on every rank over 1/N of the design, and the
    survivors' columns are gathered device to device to rank 0 for the solve
    (sharded.run_path_sharded).  Total work is fixed: "strong"."""
    ws, rank, local = _dist()
    import paper_1505_03410_b200 as gs
    from paper_1505_03410_b200 import _lib, sharded, synth
    from paper_1505_03410_b200 import dist as D
    local = _init_ranks(ws, local)
    _lib.init_device(local)
    p = int(args.p or 1_000_000)
    lo, hi = D.shard_range(p, rank, ws)
    Xs, y, _, meta = synth.cfg2_streamed(p=p, col_range=(lo, hi))
    be = sharded.DeviceBackend(Xs, y)
    v, j = be.max_abs_correlation(y)
    lmax, _ = D.argmax_over_ranks(float(v), lo + int(j))
    grid = gs.lambda_grid(lmax, 50, float(np.log10(20.0)))
    cfg = gs.SolverConfig(epsilon=1e-5 * float(y @ y), max_passes=100_000)
    import torch
    import torch.distributed as dist

    def one_path():
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = sharded.run_path_sharded(be, y, grid, cfg, p, lo)
        torch.cuda.synchronize()
        return res, (time.perf_counter() - t0) * 1e3

    for _ in range(0 if args.quick else 1):
        one_path()
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            res, t = one_path()
            ms.append(t)
    ms_step = D.max_over_ranks(statistics.mean(ms))
    if rank == 0:
        line = {"metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": ws, "steps": args.steps,
                "warmup": 1, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64 arithmetic on f32 storage", "data": "synthetic (seeded generator, SURVEY.md §8(d))",
                "config": {"workload": "cfg2", "n": int(y.size), "p": p, "lambdas": 50, "tol": 1e-5, "rule": "gap_sphere",
                           "instance": meta},
                "parallelism": f"columns sharded over {ws} ranks; X_A gathered to rank 0 (device to device)",
                "clocks": clk.summary(),
                "timing": "host clock between barriers + device synchronisation (the path is host-driven across ranks)",
                "path": {"epochs": int(sum(s.passes_done for s in res.states)), "converged": int(res.converged.sum())}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def _spawn_ranks(args) -> int:
    """``--gpus N`` outside torchrun: relaunch this script as N ranks on one
    node (one process per GPU), the way the driver does."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=600.0,
                    help="reference arm: stop starting new full paths after this many seconds")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--p", type=int, default=None, help="column count override (cfg2 / cfg4 prefixes)")
    ap.add_argument("--problems", type=int, default=256, help="cfg4: number of bootstrap problems")
    ap.add_argument("--quick", action="store_true", help="cfg2 / cfg4: skip the warm-up steps (tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "cfg4":
        return run_cfg4(args)
    if args.config == "cfg2" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_cfg2_sharded(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
