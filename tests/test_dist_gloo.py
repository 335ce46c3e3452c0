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
