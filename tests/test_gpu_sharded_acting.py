"""Acting sharded across ranks (SURVEY.md §8(e) "acting": W envs split over G GPUs, a
theta-minus broadcast once per epoch, no per-step exchange).

* One rank (dist.ShardedActing, world 1) acting for all W samplers on the executor's
  theta-minus of each epoch reproduces the transitions, frames and episodes the device
  executor (DeviceRun, concurrent mode) appended to its replay memory, bit for bit.
* Two ranks (two processes on cuda:0, torch.distributed over gloo -- NCCL needs one GPU
  per rank) each acting for W/2 samplers, gathered to rank 0: the same replay contents,
  Q rows and episodes as one rank (row independence, pkg/tests/test_nn.py:117-124).
"""

import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

EPOCHS = 2


def _hp():
    from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams

    return HyperParams(C=64, F=4, N=200, W=8, batch_size=32, total_steps=64 * EPOCHS, capacity=2000,
                       seed=3, eval_period=0, episode_length=7, terminal_p=0.05,
                       schedule=EpsilonSchedule(1.0, 0.1, 100))


def _digest(a):
    return int.from_bytes(hashlib.blake2b(np.ascontiguousarray(a).tobytes(), digest_size=8).digest(), "little")


def _contents(mem, start):
    snap = mem.snapshot()[start:]
    return ([_digest(t.state) for t in snap], [_digest(t.next_state) for t in snap],
            [t.action for t in snap], [t.reward for t in snap], [t.terminal for t in snap])


def _executor_run():
    """The device executor's epochs: theta-minus per epoch and the appended transitions."""
    from paper_2111_01264_b200.executor import DeviceRun
    from paper_2111_01264_b200.nn import copy_into

    hp = _hp()
    r = DeviceRun(hp, use_graphs=False)
    targets = []
    for e in range(EPOCHS):
        r.flush_and_merge()
        copy_into(r.target, r.theta)
        targets.append(r.target.master.clone())
        r.run_epoch(e)
        torch.cuda.synchronize()
    r.flush_and_merge()
    return targets, _contents(r.D, hp.N), list(r.record.episodes)


def _sharded(targets, rank=0, world=1):
    from paper_2111_01264_b200.dist import ShardedActing
    from paper_2111_01264_b200.nn import QNet
    from paper_2111_01264_b200.replay import ReplayMemory

    hp = _hp()
    act = ShardedActing(hp, rank, world)
    mem = ReplayMemory(hp.capacity) if rank == 0 else None
    episodes, qrows = [], []
    for e in range(EPOCHS):
        tm = QNet.empty(hp.actions)
        tm.master.copy_(targets[e])
        act.sync_target(tm if rank == 0 else None)
        act.act_epoch(e)
        frames, rec, eps = act.gather_epoch()
        qrows.append(act.q_last.cpu().numpy())
        if rank == 0:
            episodes += ShardedActing.ingest(mem, frames, rec, eps)
    torch.cuda.synchronize()
    return (_contents(mem, 0) if rank == 0 else None), episodes, qrows, act.envs.pcg_states()


def test_one_rank_matches_device_executor():
    targets, contents, episodes = _executor_run()
    mine, eps, _, _ = _sharded(targets)
    assert mine == contents
    assert eps == episodes


def _rank(rank, world, port, targets, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = _sharded([t.cuda() for t in targets], rank, world)
    q.put((rank,) + res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_match_one_rank():
    import torch.multiprocessing as mp

    targets, _, _ = _executor_run()
    one, eps1, q1, pcg1 = _sharded(targets)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 32500 + (os.getpid() % 2000)
    cpu_targets = [t.cpu() for t in targets]
    procs = [ctx.Process(target=_rank, args=(r, 2, port, cpu_targets, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (_, two, eps2, q_r0, pcg_r0), (_, _, _, q_r1, pcg_r1) = res
    assert two == one and eps2 == eps1
    for e in range(EPOCHS):  # the last block's Q rows of each rank = slices of one rank's
        assert np.array_equal(np.concatenate([q_r0[e], q_r1[e]]), q1[e])
    assert np.array_equal(np.concatenate([pcg_r0, pcg_r1]), pcg1)
