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


class DataParallelLearner:
    """Large-minibatch learner sharded over the ranks (configs[4]).

    Every rank holds the same replay memory, theta, theta-minus and optimizer state and
    draws the same global batch (same trainer stream, replay.py:65).  Rank r takes the
    contiguous shard ``shard(B, r, G)`` of the batch, computes the SUMMED gradient of its
    shard (pq_learn_grad: online / target forward, TD target, backward), the ranks
    sum-all-reduce it over NCCL, and every rank applies the identical centered RMSProp
    (pq_rmsprop_apply).  agent.train_minibatch (agent.py:84-105) feeds the optimizer the
    summed gradient of the whole batch, so the sum of the shard sums is its semantics;
    only the fp32 summation order differs from a single-device step.
    """

    def __init__(self, theta, opt, target, memory, batch: int, gamma: float = 0.99, cfg=None,
                 rank: int = 0, world_size: int = 1, process_group=None):
        from . import _native as N
        from .nn import OptConfig, workspace

        self.N = N
        self.torch = N.require_cuda()
        self.theta, self.opt, self.target, self.memory = theta, opt, target, memory
        self.batch, self.gamma = batch, gamma
        self.cfg = cfg or OptConfig()
        self.rank, self.world_size, self.group = rank, world_size, process_group
        self.lo, self.hi = shard(batch, rank, world_size)
        self.n = self.hi - self.lo
        if self.n < 1:
            raise ValueError("every rank needs at least one sample of the global batch")
        self.ws, self.cap = workspace(self.n, theta.actions)
        self.grad = self.torch.zeros_like(theta.master)
        self.flag = self.torch.full((1,), 2**31 - 1, dtype=self.torch.int32, device="cuda")
        self.updates = 0

    def _args(self, idx_shard):
        N = self.N
        c = self.cfg
        return N.PqLearnArgs(
            theta=self.theta.struct(), opt=self.opt.struct(), theta_out=self.theta.struct(),
            opt_out=self.opt.struct(), target=self.target.struct(),
            ring=self.memory.ring.data_ptr(), records=self.memory.records.data_ptr(),
            idx=idx_shard.data_ptr(), idx_base=None, update_counter=None, ext_targets=None,
            ext_actions=None, n=self.n, actions=self.theta.actions, gamma=self.gamma,
            lr=c.learning_rate, rho=c.rho, kappa=c.kappa, nonfinite=self.flag.data_ptr(),
            grad_out=None, q_out=None, td_out=None, ws=self.ws.data_ptr(), max_batch=self.cap)

    def shard_gradient(self, idx):
        """Summed gradient of this rank's shard of the global batch idx (int64 [B])."""
        N = self.N
        a = self._args(idx[self.lo:self.hi])
        N.check(N.load().pq_learn_grad(N.C.byref(a), self.grad.data_ptr(), N.stream_ptr()),
                "learn_grad")
        return self.grad

    def apply(self, grad=None):
        N = self.N
        c = self.cfg
        g = self.grad if grad is None else grad
        N.check(N.load().pq_rmsprop_apply(self.theta.struct(), self.opt.struct(), g.data_ptr(),
                                          self.theta.actions, c.learning_rate, c.rho, c.kappa,
                                          self.flag.data_ptr(), self.updates, N.stream_ptr()),
                "rmsprop_apply")
        self.opt.step += 1
        self.updates += 1

    def step(self, idx):
        """One data-parallel update on the global batch idx (device int64 [B])."""
        self.shard_gradient(idx)
        if self.world_size > 1:
            import torch.distributed as dist

            dist.all_reduce(self.grad, op=dist.ReduceOp.SUM, group=self.group)
        self.apply()

    def check_finite(self):
        v = int(self.flag.item())
        if v != 2**31 - 1:
            raise ValueError(f"gradient contains non-finite entries (update {v})")
