"""Concurrent training + synchronized execution on one B200 (executor.py:1-637).

The reference runs W sampler threads, one trainer thread and a lock-serialized
"device" (InferenceWorker).  Here the device is real:

* acting   -- one CUDA stream replays a captured graph of lockstep blocks: batched
  Nature-CNN inference over the W current stacks with theta-minus, epsilon-greedy
  and the env step in-kernel on each sampler's own PCG64 stream
  (run_epoch_lockstep, executor.py:451-510; _sampler_step :237-249);
* training -- a second stream replays a captured graph of learner steps over the
  epoch-frozen replay memory; the epoch's C/F x B indices are drawn up front from
  the trainer stream (identical consumption to C/F successive draws of B,
  replay.py:65) and sliced by a device counter (train_one, executor.py:421-434);
* epoch barrier -- stream join, owner-major flush of the sampler buffers,
  theta-minus <- theta, theta hash (execute, executor.py:552-572).

All four modes run on the device and are deterministic.  Concurrent modes ("both",
"concurrent") act from theta-minus while the learner stream trains on the frozen replay
memory.  Non-concurrent modes ("synchronized", "standard") act from theta and, before
each lockstep block, run every blocking training event that is due (train_due,
executor.py:457-460): flush the sampler buffers into the replay memory (owner-major),
draw one minibatch from it and take one learner step (blocking_train_event,
executor.py:436-440).  The samplers' Q rows always come from one batched forward (rows
are bit-identical to single-state forwards, test_nn.py:117-124); the transaction
counters follow the reference's InferenceWorker: one batched call per block when
synchronized, one single-row call per step otherwise (executor.py:115-122).  For
"standard" with W > 1 the reference is nondeterministic (executor.py:17-23); the device
runs one legal serialisation of its train gate, the lockstep one.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as N
from .agent import HyperParams, epsilon_at
from .envs import DeviceEnvs, FrameEnvSpec
from .nn import OptState, QNet, copy_into, forward, init_network, network_sizes, theta_hash, \
    workspace
from .replay import REC_INTS, ReplayMemory, device_pcg, pcg_state_to_generator, \
    sample_indices_device

ROLE_INIT = 0
ROLE_SAMPLER = 1
ROLE_TRAINER = 2
ROLE_EVAL = 3
ROLE_PREPOP = 4
ROLE_BENCH = 5


def rng_stream(seed: int, role: int, index: int = 0) -> np.random.Generator:
    """executor.py:59-63."""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(role, index)))


def derived_seed(seed: int, role: int, index: int = 0) -> int:
    """executor.py:66-68."""
    ss = np.random.SeedSequence(seed, spawn_key=(role, index))
    return int(ss.generate_state(1, np.uint64)[0])


class InferenceWorker:
    """The prediction/training device with the reference's transaction counters
    (executor.py:71-103).  Calls are stream-ordered on the GPU instead of locked."""

    def __init__(self):
        self.single_calls = 0
        self.batched_calls = 0
        self.rows_from_target = 0
        self.rows_from_main = 0
        self.train_calls = 0

    @property
    def inference_calls(self) -> int:
        return self.single_calls + self.batched_calls

    def count_predict(self, rows: int, from_target: bool, calls: int = 1) -> None:
        if rows == 1:
            self.single_calls += calls
        else:
            self.batched_calls += calls
        if from_target:
            self.rows_from_target += rows * calls
        else:
            self.rows_from_main += rows * calls

    def predict(self, params: QNet, states, *, from_target: bool):
        q = forward(params, states)
        self.count_predict(q.shape[0], from_target)
        return q

    def train(self, fn):
        self.train_calls += 1
        return fn()


def batched_inference(params: QNet, states):
    """One forward over the W sampler states (executor.py:106-112); row-independent."""
    if np.asarray(states).ndim != 4 if not hasattr(states, "dim") else states.dim() != 4:
        raise ValueError("expected a (W, 4, 84, 84) batch of sampler states")
    return forward(params, states)


def transaction_breakdown(hp: HyperParams, steps: int) -> tuple[int, int]:
    """executor.py:115-122."""
    if steps < 1 or steps % hp.C != 0:
        raise ValueError("steps must be a positive multiple of C")
    return (steps // hp.W if hp.synchronized else steps), steps // hp.F


def transaction_count(hp: HyperParams, steps: int) -> int:
    inference, training = transaction_breakdown(hp, steps)
    return inference + training


@dataclass
class RunRecord:
    """Run products + counters; CSV format of executor.py:144-209."""

    config: dict
    seed: int
    mode: str
    evals: list = field(default_factory=list)
    episodes: list = field(default_factory=list)
    epoch_hashes: list = field(default_factory=list)
    final_hash: str = ""
    counters: dict = field(default_factory=dict)
    events: list = field(default_factory=list)
    duration_s: float = 0.0
    final_params: object = None

    def to_csv_text(self) -> str:
        lines = ["# paraq-run-record v1"]
        for k in sorted(self.config):
            lines.append(f"# config {k}={self.config[k]}")
        lines.append("step,event,value")
        for step, kind, value in self.events:
            lines.append(f"{step},{kind},{value}")
        lines.append(f"# final_theta_hash {self.final_hash}")
        for k in sorted(self.counters):
            lines.append(f"# counter {k}={self.counters[k]}")
        return "\n".join(lines) + "\n"

    def write_csv(self, path) -> None:
        with open(path, "w", newline="\n") as fh:
            fh.write(self.to_csv_text())


def config_echo(hp: HyperParams) -> dict:
    return {
        "mode": hp.mode, "workers": str(hp.W), "C": str(hp.C), "F": str(hp.F),
        "gamma": repr(hp.gamma), "N": str(hp.N), "capacity": str(hp.capacity),
        "batch_size": str(hp.batch_size), "total_steps": str(hp.total_steps),
        "eval_period": str(hp.eval_period), "eval_episodes": str(hp.eval_episodes),
        "eval_epsilon": repr(hp.eval_epsilon), "eps_start": repr(hp.schedule.start),
        "eps_end": repr(hp.schedule.end), "eps_anneal": str(hp.schedule.anneal_steps),
        "lr": repr(hp.opt.learning_rate), "rho": repr(hp.opt.rho), "kappa": repr(hp.opt.kappa),
        "seed": str(hp.seed), "env": hp.env, "hidden": str(hp.hidden),
        "latency_us": repr(hp.latency_s * 1e6), "episode_length": str(hp.episode_length),
        "state_dim": str(hp.state_dim), "action_count": str(hp.action_count),
        "terminal_p": repr(hp.terminal_p),
    }


class DeviceRun:
    """Shared state and epoch driver of one device run (executor.py:341-594)."""

    def __init__(self, hp: HyperParams, env_factory=None, sink=None, use_graphs: bool = True,
                 graph_chunk: int = 25, hash_epochs: bool = True, sequential: bool = False):
        hp.validate()
        config = config_echo(hp)
        hp = apply_env_factory(hp, env_factory)
        torch = N.require_cuda()
        # non-concurrent modes: blocking training events between lockstep blocks
        self.blocking = not hp.concurrent
        self.sequential = sequential
        self.torch = torch
        self.hp = hp
        self.sink = sink
        self.use_graphs = use_graphs
        self.graph_chunk = graph_chunk
        self.hash_epochs = hash_epochs
        self._hash_pool = None
        self._pending_hashes = []
        W, C, F, B = hp.W, hp.C, hp.F, hp.batch_size
        self.steps = C // W
        self.updates = C // F
        self.worker = InferenceWorker()
        lag = -(-3 // self.steps) + 1  # epochs of stack history an env can reference
        self.lag = lag
        # frames live in the ring once each: one per transition plus the reset frames
        # (rate 1 / mean episode length, bounded here by twice that), the epoch's worst-case
        # reservation and `lag` epochs of stack history (an overrun raises, never corrupts)
        fcap = int(hp.capacity * (1.0 + reset_rate_bound(hp))) + 2 * (lag + 3) * C + 2 * W + 1024
        self.D = ReplayMemory(hp.capacity, frame_capacity=fcap)
        prepop_env = FrameEnvSpec(derived_seed(hp.seed, ROLE_PREPOP, 1), hp.episode_length,
                                  hp.actions, hp.terminal_p)
        self.D.prepopulate(prepop_env, hp.N, rng_stream(hp.seed, ROLE_PREPOP))
        self.theta = init_network(network_sizes(hp.actions), derived_seed(hp.seed, ROLE_INIT))
        self.opt = OptState.zeros(self.theta)
        self.l2_persist = os.environ.get("PQ_L2", "0") == "1"
        self._arena = self._pack_learner_state() if self.l2_persist else None
        self.target = self.theta.copy()
        keys = [derived_seed(hp.seed, ROLE_SAMPLER, 1000 + j) for j in range(W)]
        rngs = [rng_stream(hp.seed, ROLE_SAMPLER, j) for j in range(W)]
        self.envs = DeviceEnvs(keys, rngs, self.steps)
        self.envs.compact_resets()
        first = self.D._reserve_frames(W)
        slots = torch.as_tensor([(first + j) % fcap for j in range(W)], dtype=torch.int32,
                                device="cuda")
        self.envs.reset_all(slots, self.D.ring)
        self.epoch_bases = [first]
        self.trainer_pcg = device_pcg(rng_stream(hp.seed, ROLE_TRAINER))
        self.staging = torch.full((W, self.steps, REC_INTS), -1, dtype=torch.int32, device="cuda")
        self.staged = False
        # one spare row: the pipelined target forward of the epoch's last step reads the
        # (unused) minibatch after it
        self.idx_table = torch.zeros((self.updates + 1) * B, dtype=torch.int64, device="cuda")
        # pipelined target forward (bit-identical; batch 32: 70.6 vs 71.3 us/update);
        # PQ_PIPE_TARGET=0 runs the target forward inside each step
        self.pipelined = os.environ.get("PQ_PIPE_TARGET", "1") != "0" and not self.blocking
        self.update_counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.step_counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.nonfinite = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
        self.act_ws, self.act_cap = self._own_ws(W)
        self.learn_ws, self.learn_cap = self._own_ws(B)
        # PQ_PRIO=1 runs the learner's streams (and the library's wgrad branch) at the
        # highest priority; measured slower (86.7 vs 81.2 us per update), so off
        hi = -1 if os.environ.get("PQ_PRIO", "0") == "1" else 0
        # concurrent schedule with a narrow sampler batch: the acting stream runs on an
        # 8-SM green-context partition, so the lockstep acting blocks never hold SMs the
        # learner's full-width grids are waiting for (configs[1]: 64.0k -> 66.2k env
        # frames/s, bit-identical).  PQ_ACT_SMS=k overrides (0: the whole GPU).
        env_sms = os.environ.get("PQ_ACT_SMS")
        act_sms = int(env_sms) if env_sms is not None else (
            8 if (not self.blocking and not sequential and hp.W <= 16) else 0)
        self.act_stream = None
        if act_sms > 0:
            try:
                self.act_stream = N.sm_partition_stream(act_sms)
            except N.NativeError as exc:  # no green contexts here (e.g. under MPS): whole GPU
                if env_sms is not None:
                    raise
                import warnings

                warnings.warn(f"acting stream not SM-partitioned: {exc}", RuntimeWarning)
        self.act_partitioned = self.act_stream is not None
        if self.act_stream is None:
            self.act_stream = torch.cuda.Stream()
        self.learn_stream = torch.cuda.Stream(priority=hi)
        self._persist(self.learn_stream)
        self.epoch_start = 0
        self.counters = {"dfreeze_checks": 0, "dfreeze_violations": 0,
                         "prepop_pushes": self.D.version, "flush_pushes": 0}
        self.record = RunRecord(config=config, seed=hp.seed, mode=hp.mode,
                                counters=self.counters)
        self._flushed_blocks = 0   # lockstep blocks of this epoch already flushed into D
        self._epoch_trains = 0     # blocking training events of this epoch
        self._graphs = None
        self._pipe_stale = True
        self._eval_idx = 0
        self._eval = None
        self._pending_eval = None

    def _pack_learner_state(self):
        """theta's fp32 master, its bf16 shadow and the RMSProp moments in ONE allocation,
        so one L2 access-policy window can keep the learner's parameter / optimizer traffic
        (28 B per parameter per update) in the persisting L2 set-aside (PQ_L2=1; measured no
        faster at batch 32: off by default)."""
        torch = self.torch
        th, op = self.theta, self.opt
        parts = [th.master, op.m, op.v, th.shadow]
        sizes = [(t.numel() * t.element_size() + 255) // 256 * 256 for t in parts]
        arena = torch.zeros(sum(sizes), dtype=torch.uint8, device="cuda")
        views, off = [], 0
        for t, s in zip(parts, sizes):
            nb = t.numel() * t.element_size()
            v = arena[off:off + nb].view(t.dtype)
            v.copy_(t)
            views.append(v)
            off += s
        th.master, op.m, op.v, th.shadow = views
        return arena

    def _own_ws(self, n):
        torch = self.torch
        cap = max(64, 1 << (int(n) - 1).bit_length())
        nbytes = N.load().pq_workspace_bytes(cap, self.hp.actions)
        return torch.zeros(nbytes, dtype=torch.uint8, device="cuda"), cap

    def _persist(self, stream):
        if self.l2_persist:
            N.check(N.load().pq_l2_persist(N.stream_ptr(stream), self._arena.data_ptr(),
                                           self._arena.numel(), 1.0), "l2 persist")

    # -- raw step launchers (stream-ordered, graph-capturable) ----------------------------
    def _learn_args(self):
        hp = self.hp
        th, op = self.theta, self.opt
        return N.PqLearnArgs(
            theta=th.struct(), opt=op.struct(), theta_out=th.struct(), opt_out=op.struct(),
            target=self.target.struct(), ring=self.D.ring.data_ptr(),
            records=self.D.records.data_ptr(), idx=None, idx_base=self.idx_table.data_ptr(),
            update_counter=self.update_counter.data_ptr(), ext_targets=None, ext_actions=None,
            n=hp.batch_size, actions=hp.actions, gamma=hp.gamma, lr=hp.opt.learning_rate,
            rho=hp.opt.rho, kappa=hp.opt.kappa, nonfinite=self.nonfinite.data_ptr(),
            grad_out=None, q_out=None, td_out=None, ws=self.learn_ws.data_ptr(),
            max_batch=self.learn_cap)

    @property
    def acting_params(self) -> QNet:
        """theta-minus when concurrent, theta otherwise (executor.py:455, :521)."""
        return self.target if self.hp.concurrent else self.theta

    def _act_args(self):
        hp = self.hp
        s = hp.schedule
        return N.PqActArgs(
            net=self.acting_params.struct(), envs=self.envs.struct(), ring=self.D.ring.data_ptr(),
            staging=self.staging.data_ptr(), step_counter=self.step_counter.data_ptr(),
            W=hp.W, steps=self.steps, actions=hp.actions, episode_length=hp.episode_length,
            epoch_start=0, frame_capacity=self.D.frame_capacity,
            eps_start=s.start, eps_end=s.end, eps_anneal=s.anneal_steps,
            terminal_p=hp.terminal_p, q_out=None, ws=self.act_ws.data_ptr(),
            max_batch=self.act_cap)

    def learn_step(self, stream=None):
        """One self-contained learner step on the minibatch at the step counter (the
        one-shot pq_learn_step: the target forward inside the step).  Any caller may use
        it; it leaves the epoch driver's target pipeline to be re-primed."""
        a = self._learn_args()
        N.check(N.load().pq_learn_step(N.C.byref(a), N.stream_ptr(stream)), "learn_step")
        self._pipe_stale = True

    def _epoch_step(self, stream=None):
        """The epoch driver's learner step: pipelined (the target forward of the next
        minibatch rides in this step's launches, pq_learn_step_pipelined) when enabled.
        Its target activations were primed by begin_epoch / the last pipelined step."""
        if not self.pipelined:
            return self.learn_step(stream)
        if self._pipe_stale:
            self.target_prologue(stream)
        a = self._learn_args()
        N.check(N.load().pq_learn_step_pipelined(N.C.byref(a), N.stream_ptr(stream)), "learn_step")

    def target_prologue(self, stream=None):
        """Target conv1..conv3 of the minibatch at the step counter (pipelined learner)."""
        if self.pipelined:
            a = self._learn_args()
            N.check(N.load().pq_learn_target_prologue(N.C.byref(a), N.stream_ptr(stream)), "target prologue")
            self._pipe_stale = False

    def learn_epoch(self):
        """All C/F learner steps of the epoch on the current stream."""
        for _ in range(self.updates):
            self._epoch_step()

    def act_step(self, stream=None):
        a = self._act_args()
        N.check(N.load().pq_act_step(N.C.byref(a), N.stream_ptr(stream)), "act_step")

    # -- CUDA graphs ------------------------------------------------------------------
    def _capture(self):
        """Capture graph_chunk acting blocks and graph_chunk learner steps.  The
        epoch start label is read from a device scalar, so one capture serves all
        epochs; counters slice the per-epoch tables."""
        torch = self.torch
        # one eager act + learn step configures every kernel outside capture; all
        # state they touch is snapshotted and restored
        keep = [self.theta.master, self.theta.shadow, self.opt.m, self.opt.v,
                self.update_counter, self.step_counter, self.nonfinite, self.idx_table,
                self.envs.pcg, self.envs.episode, self.envs.t, self.envs.stack,
                self.envs.ep_return, self.envs.slot_next, self.envs.ep_count,
                self.envs.actions]
        saved = [t.clone() for t in keep]
        self.idx_table.zero_()
        self.act_step()
        self._epoch_step()
        torch.cuda.synchronize()
        for t, v in zip(keep, saved):
            t.copy_(v)
        k = self.graph_chunk
        graphs = {}
        for name, fn, n in (("act", self.act_step, min(k, self.steps)),
                            ("learn", self._epoch_step, min(k, self.updates))):
            g = torch.cuda.CUDAGraph()
            # an SM-partitioned acting stream captures its own graph (kernel nodes keep
            # the partition's context)
            s = self.act_stream if (name == "act" and self.act_partitioned) else torch.cuda.Stream()
            if name == "learn":
                self._persist(s)
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for _ in range(n):
                        fn()
            graphs[name] = (g, n)
        torch.cuda.synchronize()
        for t, v in zip(keep, saved):
            t.copy_(v)
        self.target_prologue()  # the warm-up step advanced the target pipeline
        return graphs

    # -- epoch pieces -------------------------------------------------------------------
    def emit(self, step, kind, value):
        self.record.events.append((step, kind, value))
        if self.sink is not None:
            self.sink(step, kind, value)

    def flush_and_merge(self):
        """Epoch-boundary flush (executor.py:385-394): staged transitions in owner-major
        order into D, finished episodes in owner order."""
        hp = self.hp
        if not self.staged:
            return
        self.flush_transitions(self.steps)
        self.trim_frames(int(self.envs.reset_next.item()))
        counts = self.envs.ep_count.cpu().numpy()
        labels = self.envs.ep_label.cpu().numpy()
        rets = self.envs.ep_ret.cpu().numpy()
        for j in range(hp.W):
            for c in range(int(counts[j])):
                self.record.episodes.append((int(labels[j, c]), float(rets[j, c])))
                self.emit(int(labels[j, c]), "episode", repr(float(rets[j, c])))
        self.envs.ep_count.zero_()
        self.staged = False
        self._flushed_blocks = 0

    def trim_frames(self, used_end: int) -> None:
        """Return the unused tail of the epoch's frame reservation (the last one made)."""
        if not self.epoch_bases[-1] <= used_end <= self.D.frame_seq:
            raise RuntimeError("frame sequence numbers out of the epoch's reservation")
        self.D.frame_seq = used_end

    def flush_transitions(self, upto_block: int) -> None:
        """Move the staged transitions of blocks [flushed, upto_block) into D in
        owner-major order (ReplayMemory.flush, replay.py:82-93: ascending owner id, each
        buffer chronological); executor.py:379-381."""
        hp = self.hp
        k0, k1 = self._flushed_blocks, upto_block
        if k1 <= k0:
            return
        n = hp.W * (k1 - k0)
        N.check(N.load().pq_replay_flush_range(
            self.staging.data_ptr(), hp.W, self.steps, k0, k1, self.D.records.data_ptr(),
            self.D.capacity, self.D.push_count, N.stream_ptr()), "flush")
        base = self.epoch_bases[max(0, len(self.epoch_bases) - 1 - self.lag)]
        self.D._advance(n, base)
        self.D._prev = None
        self.counters["flush_pushes"] += n
        self._flushed_blocks = k1

    def blocking_train_event(self, blocks_done: int) -> None:
        """Non-concurrent training (executor.py:436-440): flush the buffered transitions,
        then one minibatch drawn from the store as it is now (replay.py:61-66) and one
        learner step; the store cannot change under it (serialised on the stream)."""
        hp = self.hp
        self.flush_transitions(blocks_done)
        u = self._epoch_trains
        B = hp.batch_size
        sample_indices_device(self.trainer_pcg, len(self.D), B, out=self.idx_table[u * B:(u + 1) * B])
        self.learn_step()
        self._epoch_trains += 1
        self.worker.train_calls += 1
        self.counters["dfreeze_checks"] += 1

    def count_epoch_predictions(self) -> None:
        """InferenceWorker counters of one epoch: C/W batched W-row predictions when
        synchronized (and always in sequential_reference, executor.py:617-618), C
        single-row ones otherwise (executor.py:88-99, :115-122)."""
        hp = self.hp
        if hp.synchronized or self.sequential:  # sequential_reference: batched (:617-618)
            self.worker.count_predict(hp.W, hp.concurrent, self.steps)
        else:
            self.worker.count_predict(1, hp.concurrent, hp.C)

    def run_blocking_epoch(self) -> None:
        """Lockstep blocks with the training events due before each block's prediction and
        the rest after the last block (run_epoch_lockstep's train_due, executor.py:457-494;
        sequential_reference, executor.py:609-633)."""
        hp = self.hp
        next_train = hp.F
        for b in range(self.steps):
            while next_train <= b * hp.W:
                self.blocking_train_event(b)
                next_train += hp.F
            self.act_block(b)
        while next_train <= hp.C:
            self.blocking_train_event(self.steps)
            next_train += hp.F

    def act_block(self, b: int) -> None:
        self.act_step()

    def begin_epoch(self, epoch: int):
        """Per-epoch tables: the trainer's C/F x B indices, each sampler's frame-slot
        reservation (2 per step: next frame + possible reset frame), counters."""
        hp = self.hp
        torch = self.torch
        self.epoch_start = epoch * hp.C
        self._epoch_trains = 0
        if not self.blocking:  # the store is frozen: the epoch's C/F draws up front
            sample_indices_device(self.trainer_pcg, len(self.D), self.updates * hp.batch_size,
                                  out=self.idx_table[: self.updates * hp.batch_size])
        # worst case reserved (a next frame and a reset frame per step), the unused tail
        # returned at the flush (trim_frames): env j's next frames at base + j * steps + b,
        # the reset frames after all of them, consecutive in (step, sampler) order
        base = self.D._reserve_frames(2 * hp.C)
        self.epoch_bases.append(base)
        self.envs.slot_next.copy_(torch.arange(hp.W, device="cuda", dtype=torch.int64) * self.steps + base)
        self.envs.reset_next.fill_(base + hp.W * self.steps)
        self.update_counter.zero_()
        self.target_prologue()  # theta-minus and the index table are this epoch's

    def run_epoch(self, epoch: int):
        hp = self.hp
        torch = self.torch
        self.begin_epoch(epoch)
        if self.blocking:
            self.run_blocking_epoch()
            self.staged = True
            self.count_epoch_predictions()
            return
        if self.use_graphs and self._graphs is None:
            self._graphs = self._capture()
        cur = torch.cuda.current_stream()
        self.act_stream.wait_stream(cur)
        self.learn_stream.wait_stream(cur)
        if self.sequential:
            # single-lane schedule (sequential_reference, executor.py:596-637): all
            # sampler blocks, then the epoch's minibatches, on one stream
            for _ in range(self.steps):
                self.act_step()
            self.learn_epoch()
        elif self.use_graphs:
            self._replay_epoch()
        else:
            with torch.cuda.stream(self.learn_stream):
                self.learn_epoch()
            with torch.cuda.stream(self.act_stream):
                for _ in range(self.steps):
                    self.act_step()
        cur.wait_stream(self.act_stream)
        cur.wait_stream(self.learn_stream)
        self.staged = True
        self.count_epoch_predictions()
        self.worker.train_calls += self.updates
        self.counters["dfreeze_checks"] += self.updates

    def _replay_epoch(self):
        """Acting and training graphs interleaved on their own streams."""
        torch = self.torch
        ga, na = self._graphs["act"]
        gl, nl = self._graphs["learn"]
        if self.steps % na or self.updates % nl:
            raise RuntimeError("graph chunk must divide the per-epoch step counts")
        # t labels come from the run-global device block counter, so the same
        # captured graph serves every epoch
        ra, rl = self.steps // na, self.updates // nl
        ia = il = 0
        while ia < ra or il < rl:
            if ia < ra:
                with torch.cuda.stream(self.act_stream):
                    ga.replay()
                ia += 1
            for _ in range(2):
                if il < rl:
                    with torch.cuda.stream(self.learn_stream):
                        gl.replay()
                    il += 1

    # -- evaluation (envs.evaluate_policy, envs.py:177-202; executor.py:396-412) ---------
    # The evaluation runs on its own stream on a snapshot of the acting parameters
    # (executor.py:401 copy_parameters), overlapped with the next epoch: CUDA-graph chunks
    # of EVAL_CHUNK single-env act steps are replayed while the epoch runs, the episode
    # count comes back through pinned memory, and steps after the last episode are no-ops
    # in the kernel (max_episodes), so the result does not depend on how many chunks were
    # enqueued.  The mean / std land in the record at the boundary's place (resolve_evals).
    # With a streaming sink the evaluation completes before the boundary's events go out.
    EVAL_CHUNK = 32

    def maybe_eval(self, boundary: int):
        hp = self.hp
        if not hp.eval_period or boundary == 0 or boundary % hp.eval_period != 0:
            return
        seed = derived_seed(hp.seed, ROLE_EVAL, self._eval_idx)
        self._eval_idx += 1
        self.resolve_evals()  # one job in flight: the snapshot and the eval env are shared
        job = self._eval_start(self.acting_params, hp.eval_epsilon, hp.eval_episodes, seed)
        if self.sink is not None:
            mean, std = self._eval_finish(job)
            self.record.evals.append((boundary, mean, std))
            self.emit(boundary, "eval_mean", repr(mean))
            self.emit(boundary, "eval_std", repr(std))
            return
        slots = (len(self.record.events), len(self.record.evals))
        self.record.events += [(boundary, "eval_mean", None), (boundary, "eval_std", None)]
        self.record.evals.append((boundary, None, None))
        self._pending_eval = (slots, boundary, job)

    def resolve_evals(self):
        """Finish the evaluation in flight and fill in its record entries."""
        if self._pending_eval is None:
            return
        (i_ev, i_e), boundary, job = self._pending_eval
        self._pending_eval = None
        mean, std = self._eval_finish(job)
        self.record.events[i_ev] = (boundary, "eval_mean", repr(mean))
        self.record.events[i_ev + 1] = (boundary, "eval_std", repr(std))
        self.record.evals[i_e] = (boundary, mean, std)

    def evaluate(self, params: QNet, epsilon: float, episodes: int, seed: int):
        """Exactly `episodes` epsilon-greedy episodes of the (persistent) eval env on one
        rng stream, single-state forwards on the GPU; mean and population std."""
        self.resolve_evals()
        return self._eval_finish(self._eval_start(params, epsilon, episodes, seed))

    def _eval_state(self, episodes: int):
        """Eval env (one sampler, episode log >= episodes), its 64-frame ring, the
        parameter snapshot, the eval stream and the pinned episode counter."""
        torch = self.torch
        hp = self.hp
        log = max(256, int(episodes))
        if self._eval is None or self._eval["envs"].steps < log:
            old = self._eval
            envs = DeviceEnvs([derived_seed(hp.seed, ROLE_EVAL, 1000)],
                              [np.random.default_rng(0)], log)
            ring = torch.zeros((64, 7056), dtype=torch.uint8, device="cuda")
            if old is None:
                envs.reset_all(torch.zeros(1, dtype=torch.int32, device="cuda"), ring)
                envs.slot_next.fill_(1)
            else:  # a longer episode log: the env carries on where it was
                torch.cuda.synchronize()
                for f in ("pcg", "episode", "t", "stack", "ep_return", "slot_next", "actions"):
                    getattr(envs, f).copy_(getattr(old["envs"], f))
                ring.copy_(old["ring"])
            ws, cap = self._own_ws(1)
            self._eval = dict(
                envs=envs, ring=ring, ws=ws, cap=cap,
                staging=torch.empty((1, log, REC_INTS), dtype=torch.int32, device="cuda"),
                counter=torch.zeros(1, dtype=torch.int32, device="cuda"),
                net=old["net"] if old else self.theta.copy(),
                stream=old["stream"] if old else torch.cuda.Stream(),
                host=torch.zeros(1, dtype=torch.int32, pin_memory=True), graphs={})
        return self._eval

    def _eval_args(self, ev, epsilon: float, episodes: int):
        hp = self.hp
        envs = ev["envs"]
        return N.PqActArgs(
            net=ev["net"].struct(), envs=envs.struct(), ring=ev["ring"].data_ptr(),
            staging=ev["staging"].data_ptr(), step_counter=ev["counter"].data_ptr(), W=1,
            steps=envs.steps, actions=hp.actions, episode_length=hp.episode_length,
            epoch_start=0, frame_capacity=64, eps_start=epsilon, eps_end=epsilon,
            eps_anneal=1, terminal_p=hp.terminal_p, q_out=None, ws=ev["ws"].data_ptr(),
            max_batch=ev["cap"], max_episodes=episodes)

    def _eval_graph(self, ev, epsilon: float, episodes: int):
        """EVAL_CHUNK act steps captured once per (epsilon, episodes); a warm-up step on
        saved state configures every kernel outside the capture."""
        key = (float(epsilon), int(episodes))
        if key not in ev["graphs"]:
            torch = self.torch
            lib = N.load()
            a = self._eval_args(ev, epsilon, episodes)
            envs = ev["envs"]
            keep = [envs.pcg, envs.episode, envs.t, envs.stack, envs.ep_return, envs.slot_next,
                    envs.ep_count, envs.ep_label, envs.ep_ret, envs.actions, ev["ring"],
                    ev["counter"]]
            torch.cuda.synchronize()
            saved = [t.clone() for t in keep]
            s = ev["stream"]
            with torch.cuda.stream(s):
                N.check(lib.pq_act_step(N.C.byref(a), N.stream_ptr(s)), "eval warm-up")
            s.synchronize()
            for t, v in zip(keep, saved):
                t.copy_(v)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for _ in range(self.EVAL_CHUNK):
                        N.check(lib.pq_act_step(N.C.byref(a), N.stream_ptr(s)), "eval step")
            torch.cuda.synchronize()
            ev["graphs"][key] = (g, a)
        return ev["graphs"][key][0]

    def _eval_start(self, params: QNet, epsilon: float, episodes: int, seed: int):
        torch = self.torch
        from .replay import pcg_state_from_generator

        ev = self._eval_state(episodes)
        g = self._eval_graph(ev, epsilon, episodes)
        envs = ev["envs"]
        # snapshot + rng on the current stream (in order with the epoch that follows)
        copy_into(ev["net"], params)
        envs.pcg.copy_(torch.from_numpy(
            pcg_state_from_generator(np.random.default_rng(seed)).view(np.int64)[None]).cuda())
        envs.ep_count.zero_()
        ev["host"].zero_()
        ev["stream"].wait_stream(torch.cuda.current_stream())
        job = dict(ev=ev, graph=g, episodes=int(episodes), inflight=[], done=False)
        self._eval_pump(job)
        return job

    def _eval_chunk(self, job):
        torch = self.torch
        ev = job["ev"]
        with torch.cuda.stream(ev["stream"]):
            job["graph"].replay()
            ev["host"].copy_(ev["envs"].ep_count, non_blocking=True)
            e = torch.cuda.Event()
            e.record()
        job["inflight"].append(e)

    def _eval_pump(self, job) -> bool:
        """Keep up to two chunks in flight until the episode count (pinned, possibly
        stale) reaches the target; never blocks."""
        if job["done"]:
            return True
        inflight = job["inflight"]
        while inflight and inflight[0].query():
            inflight.pop(0)
        if int(job["ev"]["host"][0]) >= job["episodes"] and not inflight:
            job["done"] = True
            return True
        while len(inflight) < 2:
            self._eval_chunk(job)
        return False

    def _eval_finish(self, job):
        ev = job["ev"]
        while True:
            ev["stream"].synchronize()
            job["inflight"].clear()
            if int(ev["host"][0]) >= job["episodes"]:
                break
            self._eval_chunk(job)
        job["done"] = True
        rets = ev["envs"].ep_ret[0, :job["episodes"]].cpu().numpy()
        return float(rets.mean()), float(rets.std())

    def _wait_epoch(self):
        """Synchronize with the epoch just enqueued, feeding the evaluation in flight."""
        torch = self.torch
        if self._pending_eval is not None:
            done = torch.cuda.Event()
            done.record()
            job = self._pending_eval[2]
            while not done.query():
                if self._eval_pump(job):
                    break
                time.sleep(2e-4)
        torch.cuda.synchronize()

    def check_finite(self):
        v = int(self.nonfinite.item())
        if v != 2**31 - 1:
            raise ValueError(f"gradient contains non-finite entries (learner step {v} of the epoch)")

    def record_epoch_hash(self, boundary: int):
        """theta hash at an epoch boundary (executor.py:568-570).  FNV-1a is byte-serial
        (~15 ms for the 13.5 MB of f64 bytes), so without a streaming sink it runs on a
        host thread over a pinned snapshot while the next epoch runs on the GPU; its
        event keeps its place in the record (resolve_hashes, at the latest in finalize)."""
        if self.sink is not None:
            h = theta_hash(self.theta)
            self.record.epoch_hashes.append((boundary, h))
            self.emit(boundary, "theta_hash", h)
            return
        torch = self.torch
        if self._hash_pool is None:
            from concurrent.futures import ThreadPoolExecutor

            self._hash_pool = ThreadPoolExecutor(max_workers=1)
        snap = torch.empty(self.theta.master.shape, dtype=torch.float32, pin_memory=True)
        snap.copy_(self.theta.master, non_blocking=True)  # in stream order, before epoch e+1
        done = torch.cuda.Event()
        done.record()

        def work():
            done.synchronize()
            return theta_hash(snap.numpy())

        slots = (len(self.record.events), len(self.record.epoch_hashes))
        self.record.events.append((boundary, "theta_hash", None))
        self.record.epoch_hashes.append((boundary, None))
        self._pending_hashes.append((slots, boundary, self._hash_pool.submit(work)))

    def resolve_hashes(self):
        """Fill in the theta hashes still computing on the host thread."""
        for (i_ev, i_h), boundary, fut in self._pending_hashes:
            h = fut.result()
            self.record.events[i_ev] = (boundary, "theta_hash", h)
            self.record.epoch_hashes[i_h] = (boundary, h)
        self._pending_hashes.clear()

    def execute(self) -> RunRecord:
        hp = self.hp
        wall0 = time.perf_counter()
        for e in range(hp.total_steps // hp.C):
            self.flush_and_merge()
            copy_into(self.target, self.theta)
            self.maybe_eval(e * hp.C)
            self.run_epoch(e)
            self._wait_epoch()
            self.check_finite()
            if self.hash_epochs:
                self.record_epoch_hash((e + 1) * hp.C)
        self.flush_and_merge()
        self.maybe_eval(hp.total_steps)
        self.finalize(wall0)
        return self.record

    def finalize(self, wall0: float):
        self.resolve_evals()
        self.resolve_hashes()
        w = self.worker
        self.counters.update({
            "inference_single_calls": w.single_calls,
            "inference_batched_calls": w.batched_calls,
            "inference_calls": w.inference_calls,
            "acting_rows_from_target": w.rows_from_target,
            "acting_rows_from_main": w.rows_from_main,
            "train_calls": w.train_calls,
        })
        self.record.final_hash = theta_hash(self.theta)
        self.record.final_params = self.theta
        self.record.duration_s = time.perf_counter() - wall0


def reset_rate_bound(hp: HyperParams) -> float:
    """Twice the expected reset frames per env step, 1 / E[episode length] with the
    horizon L and the per-step terminal probability p: E = (1 - (1 - p)^L) / p."""
    L, p = hp.episode_length, hp.terminal_p
    mean_len = L if p <= 0 else (1.0 - (1.0 - p) ** L) / p
    return min(1.0, 2.0 / max(mean_len, 1.0))


def apply_env_factory(hp: HyperParams, env_factory) -> HyperParams:
    """The reference calls env_factory() for the prepopulation, probe, sampler and
    evaluation envs (executor.py:348-360).  Here the envs live on the device, so the
    factory must return a FrameEnvSpec: its episode_length / action_count / terminal_p
    configure every env of the run (per-role keys are derived from the seed as
    before).  None = the default env built from hp (default_env_factory, :211-218)."""
    if env_factory is None:
        return hp
    spec = env_factory()
    if not isinstance(spec, FrameEnvSpec):
        raise ValueError("env_factory must return a FrameEnvSpec: the device executor runs the "
                         f"synthetic 84x84 frame env on the GPU (got {type(spec).__name__})")
    hp = replace(hp, episode_length=int(spec.episode_length), action_count=int(spec.action_count),
                 terminal_p=float(spec.terminal_p))
    hp.validate()
    return hp


def sequential_reference(hp: HyperParams, env_factory=None, sink=None, **kw) -> RunRecord:
    """The same arithmetic as run() in one lane, canonical order: per epoch all lockstep
    blocks then the epoch's minibatches (executor.py:596-637).  The determinism oracle
    of the concurrent device executor."""
    kw.setdefault("use_graphs", False)
    return DeviceRun(hp, env_factory, sink, sequential=True, **kw).execute()


def run(hp: HyperParams, env_factory=None, sink=None, *, host_envs: bool = False,
        **kw) -> RunRecord:
    """Execute the full training run described by hp on the GPU (executor.py:591-593).
    host_envs=True keeps the samplers' envs on the CPU (end-to-end path)."""
    cls = HostEnvRun if host_envs else DeviceRun
    return cls(hp, env_factory, sink, **kw).execute()


class HostEnvRun(DeviceRun):
    """End-to-end variant: the W samplers' envs and epsilon-greedy live on the host (the
    reference's CPU sampler threads), the GPU serves batched Q-rows (InferenceWorker)
    and trains concurrently.  Every lockstep block: H2D of the current stacks' frame
    table, one batched forward on theta-minus, D2H of the W Q-rows, host select_action +
    env.step (csrc/host_env.cpp), H2D of the new frames into their ring slots.  The
    learner's graphs are enqueued for the whole epoch first and run concurrently."""

    def __init__(self, hp: HyperParams, env_factory=None, sink=None, **kw):
        super().__init__(hp, env_factory, sink, **kw)
        torch = self.torch
        W = hp.W
        lib = N.load()
        self.henv = (N.PqHenv * W)()
        for j in range(W):
            st = self.envs.pcg_states()[j]
            for k in range(6):
                self.henv[j].pcg[k] = int(st[k])
            self.henv[j].key = int(self.envs.key[j].item()) & ((1 << 64) - 1)
            self.henv[j].episode = -1
        pin = dict(pin_memory=True)
        self.h_frames = torch.empty((2 * W, 7056), dtype=torch.uint8, **pin)
        self.h_stacks = torch.empty((W, 4), dtype=torch.int32, **pin)
        self.h_q = torch.empty((W, hp.actions), dtype=torch.float32, **pin)
        self.h_staging = torch.empty((W, self.steps, REC_INTS), dtype=torch.int32, **pin)
        self.h_rec = torch.empty((W, REC_INTS), dtype=torch.int32, **pin)
        self.d_stacks = torch.empty((W, 4), dtype=torch.int32, device="cuda")
        self.d_q = torch.empty((W, hp.actions), dtype=torch.float32, device="cuda")
        self.ep_labels = np.zeros(2 * W, dtype=np.int64)
        self.ep_rets = np.zeros(2 * W, dtype=np.float64)
        self.host_episodes = [[] for _ in range(W)]
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        # initial resets (the device env state built by DeviceRun is not used)
        seq = np.array([self.D._reserve_frames(W)], dtype=np.int64)
        lib.pq_henv_reset(N.C.addressof(self.henv), W, seq.ctypes.data, self.D.frame_capacity,
                          self.h_frames.data_ptr(), self.h_stacks.data_ptr())
        self._h2d_frames(int(seq[0]) - W, W)
        torch.cuda.synchronize()

    def _h2d_frames(self, first_seq: int, count: int, stream=None):
        """Copy count new frames (consecutive sequence numbers) into their ring slots."""
        fc = self.D.frame_capacity
        s0 = first_seq % fc
        n1 = min(count, fc - s0)
        self.D.ring[s0:s0 + n1].copy_(self.h_frames[:n1], non_blocking=True)
        if n1 < count:
            self.D.ring[:count - n1].copy_(self.h_frames[n1:count], non_blocking=True)
        self.h2d_bytes += count * 7056

    def run_epoch(self, epoch: int):
        hp = self.hp
        torch = self.torch
        self.begin_epoch(epoch)
        self._seq = np.array([self.epoch_bases[-1]], dtype=np.int64)
        self._epoch = epoch
        if self.blocking:  # blocking training between the blocks, one stream
            self.run_blocking_epoch()
            self.staged = True
            self.count_epoch_predictions()
            return
        if self.use_graphs and self._graphs is None:
            self._graphs = self._capture()
        cur = torch.cuda.current_stream()
        self.act_stream.wait_stream(cur)
        self.learn_stream.wait_stream(cur)
        # the learner's whole epoch is enqueued first
        if self.use_graphs:
            gl, nl = self._graphs["learn"]
            with torch.cuda.stream(self.learn_stream):
                for _ in range(self.updates // nl):
                    gl.replay()
        else:
            with torch.cuda.stream(self.learn_stream):
                for _ in range(self.updates):
                    self._epoch_step()
        with torch.cuda.stream(self.act_stream):
            for b in range(self.steps):
                self.act_block(b)
            self.staging.copy_(self.h_staging, non_blocking=True)
            self.h2d_bytes += self.h_staging.numel() * 4
        cur.wait_stream(self.act_stream)
        cur.wait_stream(self.learn_stream)
        self.staged = True
        self.count_epoch_predictions()
        self.worker.train_calls += self.updates
        self.counters["dfreeze_checks"] += self.updates

    def act_block(self, b: int) -> None:
        """One lockstep block with host samplers on the current stream: H2D stack table,
        batched forward on the acting parameters, D2H Q-rows, host select_action + env
        step (csrc/host_env.cpp), H2D of the new frames into their ring slots."""
        hp = self.hp
        torch = self.torch
        lib = N.load()
        s = hp.schedule
        st = N.stream_ptr()
        self.d_stacks.copy_(self.h_stacks, non_blocking=True)
        self.h2d_bytes += self.h_stacks.numel() * 4
        N.check(lib.pq_forward(self.acting_params.struct(), self.D.ring.data_ptr(),
                               self.d_stacks.data_ptr(), None, 4, 0, hp.W, hp.actions,
                               self.d_q.data_ptr(), self.act_ws.data_ptr(), self.act_cap, st),
                "forward")
        self.h_q.copy_(self.d_q, non_blocking=True)
        self.d2h_bytes += self.h_q.numel() * 4
        if self._pending_eval is not None:  # feed the evaluation in flight
            self._eval_pump(self._pending_eval[2])
        torch.cuda.current_stream().synchronize()
        t_label0 = self._epoch * hp.C + b * hp.W + 1
        seq = self._seq
        first = int(seq[0])
        nf = np.zeros(1, dtype=np.int32)
        neps = np.zeros(1, dtype=np.int32)
        lib.pq_henv_step(N.C.addressof(self.henv), hp.W, self.h_q.data_ptr(), hp.actions,
                         hp.episode_length, hp.terminal_p, t_label0, s.start, s.end,
                         s.anneal_steps, seq.ctypes.data, self.D.frame_capacity,
                         self.h_frames.data_ptr(), nf.ctypes.data, self.h_stacks.data_ptr(),
                         self.h_rec.data_ptr(), self.ep_labels.ctypes.data,
                         self.ep_rets.ctypes.data, neps.ctypes.data)
        self.h_staging[:, b].copy_(self.h_rec)
        for k in range(int(neps[0])):
            lab = int(self.ep_labels[k])
            self.host_episodes[lab - t_label0].append((lab, float(self.ep_rets[k])))
        self._h2d_frames(first, int(nf[0]))

    def flush_transitions(self, upto_block: int) -> None:
        if self.blocking and upto_block > self._flushed_blocks:  # staged rows to the device
            k0 = self._flushed_blocks
            self.staging[:, k0:upto_block].copy_(self.h_staging[:, k0:upto_block], non_blocking=True)
            self.h2d_bytes += self.hp.W * (upto_block - k0) * REC_INTS * 4
        super().flush_transitions(upto_block)

    def flush_and_merge(self):
        hp = self.hp
        if not self.staged:
            return
        self.flush_transitions(self.steps)
        self.trim_frames(int(self._seq[0]))
        for j in range(hp.W):
            for lab, ret in self.host_episodes[j]:
                self.record.episodes.append((lab, ret))
                self.emit(lab, "episode", repr(ret))
            self.host_episodes[j] = []
        self.staged = False
        self._flushed_blocks = 0

    def record_epoch_hash(self, boundary: int):
        super().record_epoch_hash(boundary)
        self.d2h_bytes += self.theta.master.numel() * 4
