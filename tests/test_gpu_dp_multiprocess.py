"""Data-parallel learner across processes (configs[4]) on one GPU box.

Two ranks (both on cuda:0; torch.distributed with the gloo backend, which all-reduces
CUDA tensors through the host — NCCL needs one GPU per rank) each hold the same replay
memory and parameters, take their shard of every global batch, all-reduce the summed
shard gradients and apply the same RMSProp.  After three updates both ranks must hold
bit-identical parameters, equal to the single-process update on the full batch up to
fp32 summation order."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

B, STEPS = 512, 3


def _setup():
    from paper_2111_01264_b200 import nn as dnn
    from paper_2111_01264_b200.envs import FrameEnvSpec
    from paper_2111_01264_b200.replay import ReplayMemory, device_pcg, sample_indices_device

    mem = ReplayMemory(8192)
    mem.prepopulate(FrameEnvSpec(key=21, terminal_p=1 / 64), 6000, np.random.default_rng(3))
    theta, target = dnn.init_network(dnn.network_sizes(), 7), dnn.init_network(dnn.network_sizes(), 8)
    opt = dnn.OptState.zeros(theta)
    idx = sample_indices_device(device_pcg(np.random.default_rng(9)), len(mem), B * STEPS)
    return mem, theta, target, opt, idx


def _rank(rank, world, port, q, overlap="1"):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      PQ_DP_OVERLAP=overlap)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_01264_b200.dist import DataParallelLearner

    mem, theta, target, opt, idx = _setup()
    lr = DataParallelLearner(theta, opt, target, mem, B, rank=rank, world_size=world)
    for k in range(STEPS):
        lr.step(idx[k * B:(k + 1) * B])
    lr.check_finite()
    torch.cuda.synchronize()
    q.put((rank, theta.master.cpu().numpy(), opt.v.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _two_ranks(overlap, port):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, overlap)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_two_process_dp_learner_matches_single_process():
    from paper_2111_01264_b200.dist import DataParallelLearner

    port = 31500 + (os.getpid() % 2000)
    res = _two_ranks("0", port)
    # the bucketed all-reduce overlapped with the conv backward (the NCCL default; forced
    # here over gloo): the same sums, so bit-identical parameters
    res_ov = _two_ranks("force", port + 1)
    assert all(np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]) for a, b in zip(res, res_ov))
    (_, th0, v0), (_, th1, v1) = res
    assert np.array_equal(th0, th1) and np.array_equal(v0, v1)   # identical replicas
    mem, theta, target, opt, idx = _setup()
    single = DataParallelLearner(theta, opt, target, mem, B)   # one rank, full batch
    th_init = theta.master.cpu().numpy().copy()
    for k in range(STEPS):
        single.step(idx[k * B:(k + 1) * B])
    ref = theta.master.cpu().numpy()
    d_ref, d_dp = ref - th_init, th0 - th_init
    assert np.linalg.norm(d_dp - d_ref) / np.linalg.norm(d_ref) < 1e-3
