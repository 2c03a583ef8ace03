"""Multi-GPU plumbing for the shardable parts of the hot path.

* agent replicas (configs[3]): one independent agent per rank with a distinct seed,
  no data-path collective; job throughput = all ranks' frames / max-over-ranks time.
* large-minibatch learner (configs[4]): the batch is split into contiguous per-rank
  slices drawn from the same index stream; the per-rank summed gradients are
  all-reduced (sum) -- the reference optimizer consumes the summed gradient
  (agent.py:103-104), so a sum all-reduce of shard sums is the exact semantics.
"""

from __future__ import annotations

import os

from .executor import ROLE_BENCH, derived_seed


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def replica_seed(seed: int, rank: int) -> int:
    """Seed of agent replica `rank` (harness.py:109 convention, derived_seed ROLE_BENCH)."""
    return derived_seed(seed, ROLE_BENCH, rank) % (2**31)


def shard(batch: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of a global batch for one rank (sizes differ by <= 1)."""
    lo = batch * rank // world_size
    hi = batch * (rank + 1) // world_size
    return lo, hi


def reduce_max(value: float, device=None) -> float:
    """Max over ranks (timing: a job is as slow as its slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum_(tensor) -> None:
    """In-place sum all-reduce of a gradient shard (NCCL on GPUs, gloo in tests)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM)
