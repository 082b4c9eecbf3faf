"""Multi-GPU sharding of a batch by env index.

Envs are independent: GPU g of G owns the contiguous block
[base, base + n) of a global batch of n_total envs and uses GLOBAL indices
for its reset streams (split(from_seed(seed), base + i), batch.py:81-85) and
policy counters (step * n_total + base + i, batch.py:150-152), so env i's
trajectory is identical for any G. Nothing crosses GPUs on the hot path; the
only collective is the optional episode-statistics reduction below (a few
scalars per report interval, NCCL over NVLink on GPUs, gloo in CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    base: int      # first global env index owned by this rank
    n: int         # envs owned by this rank
    n_total: int   # envs in the whole (global) batch


def shard_range(n_total: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced split: the first n_total % world ranks get one
    extra env."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_total < world:
        raise ValueError(f"{n_total} envs cannot be split over {world} ranks")
    q, r = divmod(n_total, world)
    n = q + (1 if rank < r else 0)
    base = rank * q + min(rank, r)
    return Shard(rank=rank, world=world, base=base, n=n, n_total=n_total)


STAT_FIELDS = ("reward_sum", "episodes_done", "env_steps")


def reduce_episode_stats(stats: dict, group=None, device=None) -> dict:
    """All-reduce (sum) the per-rank episode statistics
    [reward_sum, episodes_done, env_steps]. Uses the default process group
    (NCCL on GPUs); returns the global totals. With torch.distributed not
    initialised, returns the local values."""
    import torch
    import torch.distributed as dist
    vec = torch.tensor([float(stats.get(k, 0.0)) for k in STAT_FIELDS], dtype=torch.float64,
                       device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
    return {k: float(v) for k, v in zip(STAT_FIELDS, vec.cpu().tolist())}
