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

    def buckets(self):
        """All-reduce buckets in completion order: the fc1 weight gradient (ready when its
        GEMM on the weight-gradient branch ends, 95% of the bytes), then the rest (conv
        layers, written by the last gradient kernel, and the fc1 bias / fc2 tail)."""
        from .nn import layer_shapes

        shapes = layer_shapes(self.theta.actions)
        p_w4 = sum(o * i + o for o, i in shapes[:3])
        p_b4 = p_w4 + shapes[3][0] * shapes[3][1]
        g = self.grad
        return g[p_w4:p_b4], (g[:p_w4], g[p_b4:])

    def _overlap(self) -> bool:
        """Bucketed all-reduce overlapped with the backward: NCCL by default; PQ_DP_OVERLAP=0
        turns it off, =force also takes it over gloo (the two-process test on one GPU)."""
        import torch.distributed as dist

        mode = os.environ.get("PQ_DP_OVERLAP", "1")
        return mode == "force" or (mode != "0" and dist.get_backend(self.group) == "nccl")

    def step(self, idx):
        """One data-parallel update on the global batch idx (device int64 [B]).  Over NCCL
        the fc1 weight-gradient bucket is all-reduced on a communication stream as soon as
        its GEMM completes, under the conv layers' backward; the small rest follows the
        last gradient kernel; RMSProp waits for both (PQ_DP_OVERLAP=0: one all-reduce of
        the whole gradient after it)."""
        if self.world_size == 1:
            self.shard_gradient(idx)
            self.apply()
            return
        import torch.distributed as dist

        torch, N = self.torch, self.N
        if not self._overlap():
            self.shard_gradient(idx)
            dist.all_reduce(self.grad, op=dist.ReduceOp.SUM, group=self.group)
            self.apply()
            return
        if not hasattr(self, "_comm"):
            self._comm = torch.cuda.Stream()
            self._fc1_done = torch.cuda.Event()
            self._fc1_done.record()  # creates the CUDA event handle the library records
        a = self._args(idx[self.lo:self.hi])
        N.check(N.load().pq_learn_grad_ev(N.C.byref(a), self.grad.data_ptr(), N.stream_ptr(),
                                          N.C.c_void_p(self._fc1_done.cuda_event)), "learn_grad")
        big, rest = self.buckets()
        self._comm.wait_event(self._fc1_done)
        with torch.cuda.stream(self._comm):
            w_big = dist.all_reduce(big, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        w_rest = [dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group, async_op=True) for t in rest]
        for w in [w_big] + w_rest:
            w.wait()  # the current stream waits for the collective
        self.apply()

    def check_finite(self):
        v = int(self.flag.item())
        if v != 2**31 - 1:
            raise ValueError(f"gradient contains non-finite entries (update {v})")


# ---------------------------------------------------------------- sharded acting
def pack_epoch(ring, hist, epoch_slots, staging):
    """One rank's epoch of acting as a self-contained block (pure torch; any device):
    frames = [the stack history at the epoch start (4 per sampler, zeros where masked),
    the epoch's reserved frame slots]; records = the staged [Wl, steps, 8] transitions
    with their 5 frame slots renumbered into that block (-1 stays -1)."""
    import torch

    Wl = hist.shape[0]
    fcap = ring.shape[0]
    hflat = hist.reshape(-1).long()
    nh = hflat.numel()
    lut = torch.full((fcap,), -1, dtype=torch.int64, device=ring.device)
    valid = hflat >= 0
    lut[hflat[valid]] = torch.arange(nh, device=ring.device)[valid]
    lut[epoch_slots.long()] = nh + torch.arange(epoch_slots.numel(), device=ring.device)
    frames = torch.zeros((nh + epoch_slots.numel(), ring.shape[1]), dtype=ring.dtype, device=ring.device)
    frames[:nh][valid] = ring[hflat[valid]]
    frames[nh:] = ring[epoch_slots.long()]
    rec = staging.clone()
    s = rec[..., :5].long()
    rec[..., :5] = torch.where(s >= 0, lut[s.clamp(min=0)], torch.full_like(s, -1)).to(rec.dtype)
    assert Wl == staging.shape[0]
    return frames, rec


def remap_gathered(records, frames_per_rank: int, first_seq: int, frame_capacity: int):
    """Gathered per-rank records [G, Wl, steps, 8] (slots local to each rank's block) ->
    [G*Wl, steps, 8] in global sampler order with slots into a ring where rank g's block
    starts at sequence number first_seq + g * frames_per_rank (pure torch)."""
    import torch

    G = records.shape[0]
    rec = records.clone()
    s = rec[..., :5].long()
    off = (first_seq + torch.arange(G, device=rec.device) * frames_per_rank).view(G, 1, 1, 1)
    rec[..., :5] = torch.where(s >= 0, (s + off) % frame_capacity, torch.full_like(s, -1)).to(rec.dtype)
    return rec.reshape(G * records.shape[1], records.shape[2], records.shape[3])


class ShardedActing:
    """Synchronized acting split across ranks (SURVEY.md §8(e), configs[2] / [1]): rank r
    hosts samplers shard(W, r, G) -- their device envs, PCG64 streams and frames -- and a
    theta-minus replica broadcast from rank 0 once per epoch; every lockstep block runs the
    batched Q inference + epsilon-greedy + env step of its samplers only (row
    independence, test_nn.py:117-124: Q rows do not depend on the batch), with the
    global t-labels of the unsharded schedule (executor.py:488).  At the epoch boundary
    the ranks' transitions and frames are gathered to rank 0, which appends them to its
    replay memory in ascending global owner order (replay.py:82-93) -- bit-identical to
    one GPU acting for all W samplers.  No per-block collective."""

    def __init__(self, hp, rank: int = 0, world_size: int = 1, process_group=None):
        from . import _native as N
        from .envs import DeviceEnvs
        from .executor import ROLE_SAMPLER, rng_stream
        from .nn import QNet
        from .replay import REC_INTS

        hp.validate()
        if hp.W % world_size:
            raise ValueError("W must be a multiple of the number of ranks")
        self.N, self.torch = N, N.require_cuda()
        torch = self.torch
        self.hp, self.rank, self.world_size, self.group = hp, rank, world_size, process_group
        self.lo, self.hi = shard(hp.W, rank, world_size)
        self.Wl = Wl = self.hi - self.lo
        self.steps = hp.C // hp.W
        self.per = 2 * self.steps  # frame slots per sampler per epoch (next + reset frame)
        lag = -(-3 // self.steps) + 1
        self.fcap = Wl * (self.per * (lag + 1) + 8) + 64
        self.ring = torch.zeros((self.fcap, 7056), dtype=torch.uint8, device="cuda")
        keys = [derived_seed(hp.seed, ROLE_SAMPLER, 1000 + j) for j in range(self.lo, self.hi)]
        rngs = [rng_stream(hp.seed, ROLE_SAMPLER, j) for j in range(self.lo, self.hi)]
        self.envs = DeviceEnvs(keys, rngs, self.steps)
        self.envs.reset_all(torch.arange(Wl, dtype=torch.int32, device="cuda"), self.ring)
        self.seq = Wl
        self.target = QNet.empty(hp.actions)
        self.staging = torch.full((Wl, self.steps, REC_INTS), -1, dtype=torch.int32, device="cuda")
        self.counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        cap = max(64, 1 << (Wl - 1).bit_length())
        self.ws = torch.zeros(N.load().pq_workspace_bytes(cap, hp.actions), dtype=torch.uint8, device="cuda")
        self.ws_cap = cap
        self.q_last = torch.zeros((Wl, hp.actions), dtype=torch.float32, device="cuda")
        self.epoch = 0

    def _dist(self):
        import torch.distributed as dist

        return dist if (self.world_size > 1 and dist.is_available() and dist.is_initialized()) else None

    def sync_target(self, theta_minus=None) -> None:
        """theta-minus <- rank 0's parameters (ncclBroadcast of the fp32 master once per
        epoch, executor.py:557-559), then the bf16 GEMM shadow."""
        dist = self._dist()
        if self.rank == 0:
            self.target.master.copy_(theta_minus.master)
        if dist:
            if dist.get_backend(self.group) == "gloo":
                buf = self.target.master.cpu()
                dist.broadcast(buf, 0, group=self.group)
                self.target.master.copy_(buf)
            else:
                dist.broadcast(self.target.master, 0, group=self.group)
        self.target.sync_shadow()

    def act_epoch(self, epoch: int) -> None:
        """The epoch's C/W lockstep blocks for this rank's samplers."""
        torch, N, hp = self.torch, self.N, self.hp
        self.epoch = epoch
        self.hist = self.envs.stack.clone()
        self.base = self.seq
        self.seq += self.Wl * self.per
        self.envs.slot_next.copy_(torch.arange(self.Wl, device="cuda", dtype=torch.int64) * self.per + self.base)
        self.envs.ep_count.zero_()
        s = hp.schedule
        a = N.PqActArgs(
            net=self.target.struct(), envs=self.envs.struct(), ring=self.ring.data_ptr(),
            staging=self.staging.data_ptr(), step_counter=self.counter.data_ptr(), W=self.Wl,
            steps=self.steps, actions=hp.actions, episode_length=hp.episode_length, epoch_start=0,
            frame_capacity=self.fcap, eps_start=s.start, eps_end=s.end, eps_anneal=s.anneal_steps,
            terminal_p=hp.terminal_p, q_out=self.q_last.data_ptr(), ws=self.ws.data_ptr(),
            max_batch=self.ws_cap, max_episodes=0, sampler0=self.lo, W_total=hp.W)
        for _ in range(self.steps):
            N.check(N.load().pq_act_step(N.C.byref(a), N.stream_ptr()), "act_step")

    def gather_epoch(self):
        """All ranks' epoch blocks at every rank (all_gather; rank 0 consumes them):
        frames [G, 4Wl + 2C/G, 7056], records [G, Wl, steps, 8], episodes."""
        torch = self.torch
        slots = (self.base + torch.arange(self.Wl * self.per, device="cuda")) % self.fcap
        frames, rec = pack_epoch(self.ring, self.hist, slots, self.staging)
        eps = torch.stack([self.envs.ep_count.to(torch.float64).unsqueeze(1).expand(-1, self.steps),
                           self.envs.ep_label.to(torch.float64), self.envs.ep_ret], dim=-1)
        dist = self._dist()
        if not dist:
            return frames[None], rec[None], eps[None]
        out = []
        for x in (frames, rec, eps):
            if dist.get_backend(self.group) == "gloo":
                parts = [torch.empty_like(x.cpu()) for _ in range(self.world_size)]
                dist.all_gather(parts, x.cpu(), group=self.group)
                out.append(torch.stack(parts).to(x.device))
            else:
                y = torch.empty((self.world_size,) + tuple(x.shape), dtype=x.dtype, device=x.device)
                dist.all_gather_into_tensor(y, x.contiguous(), group=self.group)
                out.append(y)
        return tuple(out)

    @staticmethod
    def ingest(memory, frames, records, episodes=None):
        """Rank 0: append the gathered epoch to the replay memory -- frames into freshly
        reserved ring slots, records renumbered and flushed owner-major (global sampler
        order = rank-major order of the contiguous shards).  Returns the finished episodes
        [(t_label, return)] in owner order (executor.py:385-394)."""
        from . import _native as N

        G, Fr = frames.shape[0], frames.shape[1]
        total = G * Fr
        first = memory._reserve_frames(total)
        torch = N.require_cuda()
        slots = (first + torch.arange(total, device="cuda")) % memory.frame_capacity
        memory.ring.index_copy_(0, slots, frames.reshape(total, -1))
        rec = remap_gathered(records, Fr, first, memory.frame_capacity).contiguous()
        W, steps = rec.shape[0], rec.shape[1]
        N.check(N.load().pq_replay_flush_range(rec.data_ptr(), W, steps, 0, steps, memory.records.data_ptr(),
                                               memory.capacity, memory.push_count, N.stream_ptr()), "flush")
        memory._advance(W * steps, first)
        memory._prev = None
        out = []
        if episodes is not None:
            e = episodes.reshape(W, steps, 3).cpu().numpy()
            for j in range(W):
                for c in range(int(e[j, 0, 0])):
                    out.append((int(e[j, c, 1]), float(e[j, c, 2])))
        return out
