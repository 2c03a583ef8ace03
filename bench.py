"""Benchmark of the fast-DQN hot path (BASELINE.json metric: env frames/sec + learner
updates/sec at batch 32).

Workload (BASELINE.json configs[1]): Nature-CNN DQN on synthetic 84x84x4 uint8
frames, 18 actions, W = 8 synchronized envs, batch 32, F = 4, 1M-transition replay
memory resident in HBM (prefilled by device prepopulation before timing), concurrent
training, target sync every C = 10,000 steps.  One bench step = one epoch: C env
frames (C/W lockstep acting blocks on one stream) + C/F learner updates (second
stream) + the epoch barrier (flush, theta-minus sync, theta hash).

  python bench.py [--gpus N --steps K --warmup W]          # the B200 arm
  python bench.py --impl reference [...]                    # the CPU reference arm

Multi-GPU (torchrun, one rank per GPU): independent agent replicas (configs[3]),
distinct seeds, no data-path collective ("replicas only" / weak scaling); the job
value is all ranks' frames over the max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env frames/sec + learner updates/sec (batch 32)"
UNIT = "env frames/s"
FLOP_PER_SAMPLE_LEARN = 68.26e6
FLOP_PER_STATE_ACT = 18.70e6
GATHER_NCU_BYTES = 2_755_831_552 + 4_460_498_432  # ncu dram bytes of the 80k gather (r2_gather_ncu.csv)
LEARN_BYTES_PER_STEP = 28 * 1_693_362  # centered RMSProp traffic of one update
GATHER_BYTES_PER_TRANSITION = 91_728  # 5 unique frames read + 8 written


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--capacity", type=int, default=1_000_000)
    ap.add_argument("--prefill", type=int, default=1_000_000)
    ap.add_argument("--C", type=int, default=10_000)
    ap.add_argument("--W", type=int, default=8)
    ap.add_argument("--B", type=int, default=32)
    ap.add_argument("--F", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweeps", action="store_true",
                    help="skip the learner-batch / acting-W sweeps and the DP learner line items")
    ap.add_argument("--dp-batch", type=int, default=1024,
                    help="global batch of the data-parallel learner measurement (configs[4])")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), \
            d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------------------- CPU arm
def bench_config(args, world: int = 1) -> dict:
    """The `config` of both arms (same workload, same keys)."""
    return {
        "workload": "configs[1]: Nature-CNN DQN, synthetic 84x84x4 uint8 frames, 18 actions, "
                    "W=8 synchronized envs, batch 32, F=4, 1M-transition replay "
                    "(prefilled), concurrent training, target sync every 10k steps; "
                    "1 step = 1 epoch (10k frames + 2.5k updates)",
        "global_batch": args.B * world, "W": args.W, "C": args.C, "F": args.F,
        "capacity": args.capacity, "prefill": args.prefill,
        "parallelism": f"replicas x{world}" if world > 1 else "single agent",
        "l2": "inputs larger than L2 (7 GB replay ring sampled uniformly)",
    }


def cpu_sample(args, updates: int, seed: int = 0):
    """The reference's concurrent schedule on the host cores with the oracle port (the
    reference kernels restated in C, single-threaded per op like numba without
    parallel=; composed like nn.py / agent.py): W sampler threads in lockstep blocks
    behind a barrier whose action is one batched forward on theta-minus
    (run_epoch_lockstep, executor.py:451-510) and one trainer thread running `updates`
    minibatch updates concurrently (_trainer_epoch, executor.py:442-447), over a bounded
    sample of the epoch: updates x F env steps.  The oracle's kernels release the GIL
    (ctypes), so samplers and trainer overlap as the reference's threads do.
    Returns (frames/s, updates/s, seconds, sample text, threads used)."""
    import threading

    from oracle import _lib as OK
    from oracle import natcnn, replay as oreplay
    from oracle.envs import SyntheticFrameEnv

    OK.set_threads(1)
    W, F, B = args.W, args.F, args.B
    spec = natcnn.nature_cnn(18)
    theta = natcnn.init_params(spec, 1 + seed)
    target = natcnn.copy_params(theta)
    opt = natcnn.Opt.zeros(theta)
    # the replay content does not change the per-op cost: a bounded prefill (the learner
    # samples from a frozen store, replay.py:61-66)
    mem = oreplay.ReplayMemory(args.capacity)
    mem.prepopulate(SyntheticFrameEnv(3 + seed, action_count=18), 2000, np.random.default_rng(seed))
    envs = [SyntheticFrameEnv(100 + j + 1000 * seed, action_count=18) for j in range(W)]
    rngs = [np.random.default_rng(j + 1000 * seed) for j in range(W)]
    states = [e.reset(r) for e, r in zip(envs, rngs)]
    blocks = max(1, updates * F // W)
    shared = {}

    def action():
        shared["q"] = natcnn.forward(spec, target, np.stack(states))

    barrier = threading.Barrier(W, action=action)
    errors = []

    def sampler(j):
        try:
            for _ in range(blocks):
                barrier.wait()
                st = OK.pcg_state_from_generator(rngs[j])
                a = OK.select_action(st, shared["q"][j], 0.1)
                OK.pcg_state_to_generator(st, rngs[j])
                nxt, rew, done = envs[j].step(a, rngs[j])
                states[j] = envs[j].reset(rngs[j]) if done else nxt
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)
            barrier.abort()

    def trainer():
        nonlocal theta, opt
        trng = np.random.default_rng(9 + seed)
        try:
            for _ in range(updates):
                batch = oreplay.gather(mem.sample(B, trng))
                theta, opt = natcnn.train_minibatch(spec, theta, opt, batch, target, 0.99)
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=sampler, args=(j,)) for j in range(W)] + [threading.Thread(target=trainer)]
    t0 = time.perf_counter()
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    secs = time.perf_counter() - t0
    if errors:
        raise errors[0]
    frames = blocks * W
    sample = (f"{updates} learner updates (B={B}) on 1 trainer thread concurrent with {blocks} lockstep "
              f"blocks of W={W} sampler threads (batched forward on theta-minus, select_action, env step) "
              f"= {frames} env steps of the Nature-CNN oracle in {secs:.1f} s")
    return frames / secs, updates / secs, secs, sample, W + 1


def _replica_worker(args, updates, seed, q):
    q.put(cpu_sample(args, updates, seed)[:3])


def cpu_replicas(args, updates: int):
    """configs[3] on the host: independent agent replicas as processes,
    as many as the cores hold W sampler + 1 trainer threads each; aggregate frames/s."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    n = max(1, min(8, cores // (args.W + 1)))
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_replica_worker, args=(args, updates, k + 1, q)) for k in range(n)]
    t0 = time.perf_counter()
    for p in procs:
        p.start()
    res = [q.get() for _ in procs]
    for p in procs:
        p.join()
    wall = time.perf_counter() - t0
    frames = sum(r[0] * r[2] for r in res)
    return {"replicas": n, "threads_per_replica": args.W + 1, "frames_per_s": frames / wall,
            "updates_per_s": sum(r[1] * r[2] for r in res) / wall, "wall_s": wall}


def run_reference(args, rank: int):
    """--impl reference: the reference's CPU path (the oracle port, this tier's reference
    arm) on the box's host cores in the reference's own thread model; each step is a
    bounded sample of the configs[1] epoch (UPD updates with their F x UPD env steps)."""
    if rank != 0:
        return
    upd = int(os.environ.get("PQ_REF_UPDATES", "4"))
    vals, ups, secs = [], [], []
    sample, used = "", 0
    for k in range(args.warmup + args.steps):
        fs, us, s, sample, used = cpu_sample(args, upd, seed=k)
        if k >= args.warmup:
            vals.append(fs), ups.append(us), secs.append(s)
    value = float(np.median(vals))
    updates_s = float(np.median(ups))
    full_updates = 50_000 // args.F  # configs[0]: a 50k-step run (SURVEY §8(d) runs > 1 h)
    reps = cpu_replicas(args, upd) if os.environ.get("PQ_REF_REPLICAS", "1") == "1" else None
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * float(np.median(secs)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "learner_updates_per_s": updates_s,
        "config": bench_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "port",
                         "sample": sample + f" (one step = one such sample; median of {args.steps})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolation": {"full_run": "configs[0]: 50k env steps, 12,500 updates",
                          "seconds": full_updates / updates_s, "hours": full_updates / updates_s / 3600,
                          "note": "extrapolated from the measured update rate, printed beside the "
                                  "measurement (harness.py:410-426), never substituted"},
        "cpu_replicas": reps,
        "host_cores": len(os.sched_getaffinity(0)),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 arm
def time_learner_graph(runner, epoch: int):
    """Average device time of one learner step as the bench runs it: one epoch's worth
    of replays of the captured learner graph (the PDL-chained launches) on the learner
    stream, CUDA events on that stream; learner state restored afterwards."""
    import torch

    gl, nl = runner._graphs["learn"]
    keep = (runner.theta.master, runner.theta.shadow, runner.opt.m, runner.opt.v, runner.update_counter)
    saved = [t.clone() for t in keep]
    runner.begin_epoch(epoch)
    ls = runner.learn_stream
    ls.wait_stream(torch.cuda.current_stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ls):
        e0.record(ls)
        for _ in range(runner.updates // nl):
            gl.replay()
        e1.record(ls)
    torch.cuda.synchronize()
    learn_ms = e0.elapsed_time(e1) / (runner.updates // nl * nl)
    for t, v in zip(keep, saved):
        t.copy_(v)
    torch.cuda.synchronize()
    return learn_ms


def time_gather(runner, transitions: int = 80_000, reps: int = 10):
    """Replay sample + stack gather over an epoch-sized batch (HBM-bound), per engine:
    {"tma": ms, "ldg": ms} (pq_replay_gather runs the 16-byte-load one)."""
    import torch
    from paper_2111_01264_b200.replay import device_pcg, sample_indices_device

    st = device_pcg(np.random.default_rng(123))
    idx = sample_indices_device(st, len(runner.D), transitions)
    B = transitions
    s = torch.empty((B, 4, 84, 84), dtype=torch.uint8, device="cuda")
    s2 = torch.empty_like(s)
    a = torch.empty(B, dtype=torch.int32, device="cuda")
    r = torch.empty(B, dtype=torch.float64, device="cuda")
    t = torch.empty(B, dtype=torch.uint8, device="cuda")
    from paper_2111_01264_b200 import _native as N

    lib = N.load()
    out = {}
    for name, fn in (("tma", lib.pq_replay_gather_tma), ("ldg", lib.pq_replay_gather_ldg)):
        def go():
            N.check(fn(runner.D.ring.data_ptr(), runner.D.records.data_ptr(), idx.data_ptr(), B, s.data_ptr(),
                       s2.data_ptr(), a.data_ptr(), r.data_ptr(), t.data_ptr(), N.stream_ptr()), "gather")
        go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            go()
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    del s, s2
    return out


def learner_sweep(memory, actions: int, batches=(32, 64, 128, 256, 512, 1024), steps: int = 40):
    """configs[4] sizes on one GPU: learner updates/s of the one-shot tcgen05 learner step
    (eager launches, theta / opt updated in place) at each batch, and the achieved
    tensor-core rate over the step (68.26 MFLOP per sample)."""
    import ctypes

    import torch
    from paper_2111_01264_b200 import _native as N
    from paper_2111_01264_b200 import nn as dnn

    lib = N.load()
    out = []
    for B in batches:
        theta = dnn.init_network(dnn.network_sizes(actions), 1)
        target = dnn.init_network(dnn.network_sizes(actions), 2)
        opt = dnn.OptState.zeros(theta)
        ws, cap = dnn.workspace(B, actions)
        flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
        idx = torch.as_tensor(memory.sample_indices(B * (steps + 5), np.random.default_rng(B)), device="cuda")
        a = N.PqLearnArgs(theta=theta.struct(), opt=opt.struct(), theta_out=theta.struct(), opt_out=opt.struct(),
                          target=target.struct(), ring=memory.ring.data_ptr(), records=memory.records.data_ptr(),
                          idx=None, idx_base=None, update_counter=None, ext_targets=None, ext_actions=None,
                          n=B, actions=actions, gamma=0.99, lr=2.5e-4, rho=0.95, kappa=0.01,
                          nonfinite=flag.data_ptr(), grad_out=None, q_out=None, td_out=None,
                          ws=ws.data_ptr(), max_batch=cap)
        st = N.stream_ptr()

        def go(k):
            a.idx = idx[k * B:(k + 1) * B].data_ptr()
            N.check(lib.pq_learn_step(ctypes.byref(a), st), "learn_step")

        for k in range(5):
            go(steps + k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(steps):
            go(k)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out.append({"batch": B, "updates_per_s": 1e3 / ms, "us_per_update": ms * 1e3,
                    "tflops": FLOP_PER_SAMPLE_LEARN * B / (ms * 1e-3) / 1e12})
    return out


def act_sweep(actions: int, widths=(8, 32, 128, 512), reps: int = 50):
    """configs[2]: batched Q inference over W synchronized env states (nn.forward on
    theta-minus, tcgen05 conv/fc GEMMs + head): states/s and tensor-core rate
    (18.70 MFLOP per state).  The env step / epsilon-greedy kernel is measured inside
    the epoch bench (k_act_env)."""
    import torch
    from paper_2111_01264_b200 import _native as N
    from paper_2111_01264_b200 import nn as dnn

    lib = N.load()
    net = dnn.init_network(dnn.network_sizes(actions), 3)
    out = []
    for W in widths:
        ring = torch.randint(0, 256, (4 * W, 84 * 84), dtype=torch.uint8, device="cuda")
        refs = torch.arange(4 * W, dtype=torch.int32, device="cuda").view(W, 4)
        q = torch.empty((W, actions), dtype=torch.float32, device="cuda")
        ws, cap = dnn.workspace(W, actions)

        def go():
            N.check(lib.pq_forward(net.struct(), ring.data_ptr(), refs.data_ptr(), None, 4, 0, W, actions,
                                   q.data_ptr(), ws.data_ptr(), cap, N.stream_ptr()), "forward")

        for _ in range(5):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            go()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out.append({"W": W, "us_per_block": ms * 1e3, "states_per_s": W / (ms * 1e-3),
                    "tflops": FLOP_PER_STATE_ACT * W / (ms * 1e-3) / 1e12})
    return out


def sharded_acting(args, rank: int, world: int, dist, per_rank: int = 512, blocks: int = 20, epochs: int = 2):
    """configs[2] acting sharded over the ranks (dist.ShardedActing): each rank
    hosts per_rank synchronized envs (W = per_rank x ranks, weak scaling) and runs the
    epoch's lockstep blocks (batched Q inference + epsilon-greedy + env step); per epoch a
    theta-minus broadcast from rank 0 and an all-gather of the epoch's frames and records,
    which rank 0 appends to its replay memory.  Env steps/s over all ranks, timed on the
    device, max over ranks, collectives and the ingest included."""
    import torch
    from paper_2111_01264_b200 import nn as dnn
    from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
    from paper_2111_01264_b200.dist import ShardedActing
    from paper_2111_01264_b200.replay import ReplayMemory

    W = per_rank * world
    C = W * blocks
    hp = HyperParams(C=C, F=4, N=0, W=W, batch_size=32, total_steps=C, capacity=4 * C, seed=args.seed,
                     eval_period=0, schedule=EpsilonSchedule(0.1, 0.1, 1))
    act = ShardedActing(hp, rank, world)
    theta = dnn.init_network(dnn.network_sizes(hp.actions), 11) if rank == 0 else None
    mem = ReplayMemory(4 * C, frame_capacity=3 * world * (4 * per_rank + 2 * C // world) + 1024) if rank == 0 else None

    def epoch(e):
        act.sync_target(theta)
        act.act_epoch(e)
        fr, rec, eps = act.gather_epoch()
        if rank == 0:
            ShardedActing.ingest(mem, fr, rec)

    epoch(0)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for e in range(1, 1 + epochs):
        epoch(e)
    e1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    steps = epochs * C
    return {"W_total": W, "per_rank_envs": per_rank, "ranks": world, "blocks_per_epoch": blocks,
            "env_steps_per_s": steps / (ms * 1e-3), "us_per_block": ms * 1e3 / (epochs * blocks),
            "q_inference_tflops": FLOP_PER_STATE_ACT * steps / (ms * 1e-3) / 1e12,
            "scaling": "weak",
            "collective": ("theta-minus broadcast + all-gather of the epoch's frames / records per epoch "
                           f"({dist.get_backend()})") if dist else "none (1 rank)"}


def dp_learner(args, rank: int, world: int, dist, steps: int = 30):
    """configs[4] across ranks: global batch args.dp_batch split over the ranks, shard
    gradients sum-all-reduced over NCCL, identical RMSProp everywhere (dist.py).  All
    ranks hold the same 100k-transition replay memory (same prepopulation seed) and
    draw the same indices.  Returns updates/s of the whole job (max-over-ranks time)."""
    import torch
    from paper_2111_01264_b200 import nn as dnn
    from paper_2111_01264_b200.dist import DataParallelLearner
    from paper_2111_01264_b200.envs import FrameEnvSpec
    from paper_2111_01264_b200.replay import ReplayMemory, device_pcg, sample_indices_device

    B = args.dp_batch
    mem = ReplayMemory(100_000)
    mem.prepopulate(FrameEnvSpec(key=77), 100_000, np.random.default_rng(4))
    theta = dnn.init_network(dnn.network_sizes(), 5)
    target = dnn.init_network(dnn.network_sizes(), 6)
    opt = dnn.OptState.zeros(theta)
    lr = DataParallelLearner(theta, opt, target, mem, B, rank=rank, world_size=world)
    pcg = device_pcg(np.random.default_rng(8))
    idx = sample_indices_device(pcg, len(mem), B * (steps + 3))
    for k in range(3):
        lr.step(idx[(steps + k) * B:(steps + k + 1) * B])
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(steps):
        lr.step(idx[k * B:(k + 1) * B])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    lr.check_finite()
    ups = steps / (ms / 1e3)
    return {"global_batch": B, "ranks": world, "per_rank_batch": lr.n, "updates_per_s": ups,
            "samples_per_s": ups * B, "tflops": FLOP_PER_SAMPLE_LEARN * B * ups / 1e12,
            "collective": (f"all-reduce (sum) of the 6.77 MB fp32 gradient per update over {dist.get_backend()}"
                           + (": the 6.4 MB fc1-weight bucket on a communication stream as soon as its GEMM "
                              "ends, under the conv backward, then the rest" if lr._overlap() else ""))
            if world > 1 else "none (1 rank)"}


def run_b200(args, rank: int, world: int, local_rank: int):
    import torch

    # PQ_BENCH_SHARE_GPU=1 (multi-rank smoke test on a one-GPU box only): ranks share the
    # visible devices and the collectives go over gloo; the driver's runs use one GPU per
    # rank and NCCL
    share = os.environ.get("PQ_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
    from paper_2111_01264_b200.executor import ROLE_BENCH, DeviceRun, derived_seed
    from paper_2111_01264_b200.nn import copy_into

    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    seed = derived_seed(args.seed, ROLE_BENCH, rank) % (2**31)
    total_epochs = args.warmup + args.steps
    hp = HyperParams(C=args.C, F=args.F, N=args.prefill, W=args.W, batch_size=args.B,
                     total_steps=args.C * total_epochs, capacity=args.capacity, seed=seed,
                     schedule=EpsilonSchedule(0.1, 0.1, 1), eval_period=0)
    t_setup = time.perf_counter()
    runner = DeviceRun(hp, use_graphs=True, graph_chunk=250)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    def epoch(e):
        runner.flush_and_merge()
        copy_into(runner.target, runner.theta)
        runner.run_epoch(e)
        torch.cuda.synchronize()
        runner.check_finite()
        runner.record_epoch_hash((e + 1) * hp.C)

    for e in range(args.warmup):
        epoch(e)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for e in range(args.warmup, total_epochs):
        epoch(e)
    e1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    secs = ms / 1000.0
    frames = world * args.steps * hp.C
    value = frames / secs
    updates_s = world * args.steps * (hp.C // hp.F) / secs
    # kernel-level measurements (outside the timed region; same inputs)
    learn_ms = time_learner_graph(runner, total_epochs)
    gather_ms = time_gather(runner)
    sweeps = {}
    if not args.no_sweeps and world == 1:
        sweeps["learner_batch_sweep"] = learner_sweep(runner.D, hp.actions)
        sweeps["acting_width_sweep"] = act_sweep(hp.actions)
    del runner
    torch.cuda.empty_cache()
    if not args.no_sweeps:
        # secondary keys: a failure is recorded in the line instead of losing it (the same
        # code runs on every rank, so an error is raised on all of them alike)
        def secondary(fn):
            try:
                return fn(args, rank, world, dist)
            except Exception as exc:  # noqa: BLE001
                import traceback

                traceback.print_exc()
                return {"error": f"{type(exc).__name__}: {exc}"[:300]}

        sweeps["dp_learner"] = secondary(dp_learner)
        torch.cuda.empty_cache()
        sweeps["acting_sharded"] = secondary(sharded_acting)
    torch.cuda.empty_cache()
    # end to end through the public API with host envs: H2D frames + D2H Q-rows per
    # lockstep block, theta hash D2H per epoch (the paper's CPU-env / GPU setting)
    from paper_2111_01264_b200.executor import HostEnvRun

    erun = HostEnvRun(hp, use_graphs=True, graph_chunk=250)

    def e_epoch(e):
        erun.flush_and_merge()
        copy_into(erun.target, erun.theta)
        erun.run_epoch(e)
        torch.cuda.synchronize()
        erun.check_finite()
        erun.record_epoch_hash((e + 1) * hp.C)

    for e in range(args.warmup):
        e_epoch(e)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    h2d0, d2h0 = erun.h2d_bytes, erun.d2h_bytes
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for e in range(args.warmup, total_epochs):
        e_epoch(e)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": world * args.steps * hp.C / (e2e_ms / 1000.0), "unit": UNIT,
           "h2d_bytes_per_step": (erun.h2d_bytes - h2d0) // args.steps,
           "d2h_bytes_per_step": (erun.d2h_bytes - d2h0) // args.steps,
           "path": "executor.run(host_envs=True): CPU samplers (select_action + env.step in C), "
                   "per lockstep block H2D stacks + new frames from pinned memory and D2H of the "
                   "W Q-rows; per epoch H2D staging, D2H theta for the hash"}
    del erun
    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return
    hbm, bf16_burst, bf16_sus, peak_src = measured_peaks()
    traffic, traffic_src = None, None  # DRAM bytes of one learner step (committed ncu capture)
    for name in ("r2_v5_traffic.json", "r2_v4_traffic.json", "r2_v3_traffic.json", "r2_v2_traffic.json", "r2_traffic.json",
                 "r1_traffic.json"):
        tpath = os.path.join(ROOT, "profiles", name)
        if os.path.exists(tpath):
            with open(tpath) as fh:
                traffic = json.load(fh).get("learner_step_dram_bytes")
            traffic_src = (f"profiles/{name} (ncu --set full, dram__bytes_read+write summed over one "
                           "step's launches, cold caches)")
            break
    learn_flop = FLOP_PER_SAMPLE_LEARN * hp.batch_size
    achieved_tf = learn_flop / (learn_ms * 1e-3) / 1e12
    gather_gbs = 80_000 * GATHER_BYTES_PER_TRANSITION / (gather_ms["ldg"] * 1e-3) / 1e9
    gather_tma_gbs = 80_000 * GATHER_BYTES_PER_TRANSITION / (gather_ms["tma"] * 1e-3) / 1e9
    per_epoch_launches = (hp.C // hp.W) * 5 + (hp.C // hp.F) * 10 + 5  # + flush, copy, target prologue (3)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        fs, us, s, sample, used = cpu_sample(args, int(os.environ.get("PQ_REF_UPDATES", "4")))
        cpu = {"value": fs, "unit": UNIT, "cores": used, "kind": "port", "sample": sample,
               "updates_per_s": us}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "learner_updates_per_s": updates_s,
        "config": dict(bench_config(args, world), setup_s=round(setup_s, 2)),
        "roofline": {
            "kernel": "learner step (batch 32: 10 dependent launches -- conv1..fc1 forward, head, fc1 "
                      "dgrad, 3 fused dgrad / wgrad / RMSProp grids, update)",
            "bound": "tensor", "achieved": achieved_tf, "peak": bf16_sus, "unit": "TFLOP/s",
            "frac": achieved_tf / bf16_sus, "traffic": traffic,
            "binding": "latency: a chain of 10 dependent launches of 1-9 small GEMM tiles each "
                       "(profiles/r2_v6_cta_trace_b32.txt); neither the tensor pipe nor HBM is saturated",
            "traffic_source": traffic_src,
            "per_launch": f"{learn_flop / 1e9:.3f} GFLOP (68.26 MFLOP/sample x {hp.batch_size}) "
                          f"in {learn_ms * 1e3:.1f} us",
            "peak_source": f"{peak_src}: bf16_tflops_sustained (the step is timed inside a seconds-long epoch)",
        },
        "learner_memory_floor": {
            "bound": "hbm", "algorithmic_bytes": LEARN_BYTES_PER_STEP,
            "achieved": LEARN_BYTES_PER_STEP / (learn_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": LEARN_BYTES_PER_STEP / (learn_ms * 1e-3) / 1e9 / hbm,
            "note": "28 B per parameter of centered RMSProp (read p, m, v; write p, m, v, bf16 "
                    "shadow) x 1,693,362 parameters: the step's memory floor",
        },
        "gather_roofline": {
            "kernel": "k_gather (pq_replay_gather: 16-byte vector loads; 80k-transition sample, "
                      "91,728 B each)", "bound": "hbm",
            "achieved": gather_gbs, "peak": hbm, "unit": "GB/s", "frac": gather_gbs / hbm,
            "ms": gather_ms["ldg"],
            "traffic": GATHER_NCU_BYTES, "traffic_source": "profiles/r2_gather_ncu.csv (dram__bytes_read+write "
                                                           "of the same 80k gather, ncu)",
            "tma_engine": {"kernel": "k_gather_tma (TMA bulk copies through a shared-memory ring)",
                           "ms": gather_ms["tma"], "achieved": gather_tma_gbs, "frac": gather_tma_gbs / hbm},
        },
        "gpu_launches": per_epoch_launches * args.steps,
        **sweeps,
        "clocks": clk,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
