"""World-size-2 gloo tests of the multi-process plumbing (CPU only).

Covers the N > 1 path of bench.py (max-over-ranks timing) and the
deterministic cross-rank reductions a column-sharded screening pass needs
(arg-max with smallest-index ties, rank-ordered sums)."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

from paper_1505_03410_b200.dist import shard_range  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist
    from paper_1505_03410_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        out["max"] = D.max_over_ranks(1.5 + rank)
        # column-sharded |X^T y|_inf: each rank scans its block, ties -> smallest index
        rng = np.random.default_rng(0)
        c = np.abs(rng.standard_normal(101))
        c[17] = c[80] = c.max() + 1.0           # a tie across the two shards
        lo, hi = D.shard_range(c.size, rank, world)
        loc = lo + int(np.argmax(c[lo:hi]))
        out["argmax"] = D.argmax_over_ranks(float(c[loc]), loc)
        out["argmax_ref"] = (float(c.max()), int(np.argmax(c)))
        parts = [0.1, 0.2]
        out["sum"] = D.rank_ordered_sum(parts[rank])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for total in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_gloo_world2_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert res[r]["max"] == 2.5
        assert res[r]["argmax"] == res[r]["argmax_ref"]
        assert res[r]["argmax"][1] == 17
        assert res[r]["sum"] == 0.1 + 0.2


def test_bench_reference_arm_under_torchrun_world2():
    """bench.py's N > 1 launch path on CPU: ``--gpus 2`` relaunches the script
    as two ranks (torch.distributed.run, 127.0.0.1); rank 0 alone runs the
    reference arm and prints ONE JSON line, rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "cfg0", "--p", "300", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["steps"] == 1
    assert line["config"]["workload"] == "cfg0" and line["config"]["p"] == 300
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_bench_cfg4_problem_sharded_two_ranks():
    """bench.py --config cfg4 --gpus 2 on the device: problems sharded by index
    over two ranks (sharing the GPU when the box has one; no kernel of one rank
    waits on the other), one JSON line with the parity block green."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "cfg4", "--gpus", "2",
                          "--problems", "4", "--p", "2000", "--steps", "1", "--quick", "--cpu-budget", "5"],
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["config"]["workload"] == "cfg4" and line["scaling"] == "strong"
    assert line["parity"]["ok"] and line["gpu_launches"] >= 1


@pytest.mark.gpu
def test_bench_cfg2_column_sharded_two_ranks():
    """bench.py --config cfg2 --gpus 2 on the device: column shards, X_A gathered
    device to device (gloo moves it when the ranks share one GPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "cfg2", "--gpus", "2",
                          "--p", "20000", "--steps", "1", "--quick"],
                         capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["path"]["converged"] == 50
