"""Multi-process plumbing (one process per GPU, torch.distributed).

The Lasso path shards only where SURVEY.md §8(e) says it does:
  * the full-p screening pass by contiguous column blocks (cfg2), whose
    reductions are an arg-max with smallest-index tie break (lambda_max,
    |X_A^T rho|_inf) and rank-ordered sums (||beta||_1 partials) -- both
    deterministic, unlike a floating-point all-reduce sum;
  * independent problems by index (cfg4);
  * otherwise replicas (cfg0, cfg1, cfg3).
These helpers are backend-agnostic (NCCL on the GPU box, gloo in the CPU
tests).  Timings are reduced as the max over ranks.
"""

from __future__ import annotations


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of ``total`` items owned by ``rank``; blocks
    differ in size by at most one and are ordered by rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist
    return dist


def _device():
    import torch
    dist = _dist()
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(x: float) -> float:
    import torch
    dist = _dist()
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def argmax_over_ranks(val: float, idx: int) -> tuple[float, int]:
    """Global (max value, smallest index attaining it) from per-rank
    (value, global index) pairs -- design_matrix.py:160-174 semantics."""
    import torch
    dist = _dist()
    world = dist.get_world_size()
    mine = torch.tensor([float(val), float(idx)], dtype=torch.float64, device=_device())
    out = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(out, mine)
    best_v, best_i = -1.0, None
    for t in out:
        v, i = float(t[0].item()), int(t[1].item())
        if v > best_v or (v == best_v and (best_i is None or i < best_i)):
            best_v, best_i = v, i
    return best_v, best_i


def rank_ordered_sum(x: float) -> float:
    """Sum of per-rank partials added in rank order (bit-reproducible)."""
    import torch
    dist = _dist()
    world = dist.get_world_size()
    mine = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    out = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(out, mine)
    s = 0.0
    for t in out:
        s += float(t.item())
    return s
