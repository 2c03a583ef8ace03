"""Data-parallel learner (configs[4]) on one GPU.

The DP step's semantics are checked without a second GPU: the summed gradients of the
shards of a batch ("virtual ranks" rank r of G, all on cuda:0) must add up to the
summed gradient of the whole batch, and one DP update (shard gradients summed as the
NCCL all-reduce would, then pq_rmsprop_apply) must equal the single-device learner
step (agent.train_minibatch) up to fp32 summation order.  The per-sample forward rows
are bit-identical whatever the batch composition (row independence, test_nn.py:117-124),
so only the batch reductions of the weight gradients can differ: tolerance 1e-5
relative."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2111_01264_b200 import nn as dnn  # noqa: E402
from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams  # noqa: E402
from paper_2111_01264_b200.dist import DataParallelLearner  # noqa: E402
from paper_2111_01264_b200.envs import FrameEnvSpec  # noqa: E402
from paper_2111_01264_b200.executor import DeviceRun  # noqa: E402
from paper_2111_01264_b200.replay import ReplayMemory  # noqa: E402

A = 18


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / max(b.norm(), 1e-30))


@pytest.fixture(scope="module")
def memory():
    mem = ReplayMemory(4096)
    mem.prepopulate(FrameEnvSpec(key=11, terminal_p=1 / 64), 3000, np.random.default_rng(5))
    return mem


def fresh(seed=2):
    theta = dnn.init_network(dnn.network_sizes(A), seed)
    target = dnn.init_network(dnn.network_sizes(A), seed + 1)
    return theta, dnn.OptState.zeros(theta), target


# shards and full batch on the same GEMM engine (cp.async below batch 128, TMA from 128:
# qnet.cu use_tma): the per-sample forward rows are then bit-identical
@pytest.mark.parametrize("B,G", [(64, 2), (512, 2), (1024, 8), (33, 3)])
def test_shard_gradients_sum_to_batch_gradient(memory, B, G):
    idx = torch.as_tensor(memory.sample_indices(B, np.random.default_rng(B)), device="cuda")
    theta, opt, target = fresh()
    full = DataParallelLearner(theta, opt, target, memory, B).shard_gradient(idx).clone()
    total = torch.zeros_like(full)
    for r in range(G):
        total += DataParallelLearner(theta, opt, target, memory, B, rank=r,
                                     world_size=G).shard_gradient(idx)
    assert torch.isfinite(full).all()
    assert rel(total, full) < 1e-5


def test_shard_gradients_across_engines(memory):
    """Batch 256 (TMA engine, space-to-depth conv1 with a permuted K order) against four
    batch-64 shards (cp.async engine): the fp32 accumulation orders differ, so rare bf16
    roundings of activations differ; the sum still matches to the conditioning bound of
    the stage-wise tests."""
    B, G = 256, 4
    idx = torch.as_tensor(memory.sample_indices(B, np.random.default_rng(B)), device="cuda")
    theta, opt, target = fresh()
    full = DataParallelLearner(theta, opt, target, memory, B).shard_gradient(idx).clone()
    total = torch.zeros_like(full)
    for r in range(G):
        total += DataParallelLearner(theta, opt, target, memory, B, rank=r,
                                     world_size=G).shard_gradient(idx)
    assert rel(total, full) < 2e-2


@pytest.mark.parametrize("B", [64, 512])
def test_dp_update_equals_single_device_step(memory, B):
    idx = torch.as_tensor(memory.sample_indices(B, np.random.default_rng(7)), device="cuda")
    theta, opt, target = fresh()
    ref_theta, ref_opt, _, _, _ = dnn._learn(theta, opt, target, memory.ring, memory.records, idx, B)
    G = 4
    learners = [DataParallelLearner(theta.copy(), dnn.OptState(opt.m.clone(), opt.v.clone()), target,
                                     memory, B, rank=r, world_size=G) for r in range(G)]
    grad = sum(lr.shard_gradient(idx).clone() for lr in learners)   # the NCCL sum all-reduce
    for lr in learners:
        lr.apply(grad)
        lr.check_finite()
    torch.cuda.synchronize()
    for lr in learners[1:]:   # every rank holds the identical update
        assert torch.equal(lr.theta.master, learners[0].theta.master)
    d_ref = ref_theta.master - theta.master
    assert rel(learners[0].theta.master - theta.master, d_ref) < 1e-4
    assert rel(learners[0].opt.v, ref_opt.v) < 1e-4
    # the bf16 GEMM shadow follows the master
    assert torch.equal(learners[0].theta.shadow[:8192],
                       learners[0].theta.master[:8192].bfloat16().view(torch.int16))


@pytest.mark.parametrize("B", [64, 1024])
def test_gradient_event_marks_the_fc1_bucket(memory, B):
    """pq_learn_grad_ev (the NCCL-overlapped DP step): the same gradient as pq_learn_grad,
    and when its fc1 event has fired the fc1 bucket already holds its final values even
    though the conv layers' backward may still run; the two buckets tile the gradient."""
    from paper_2111_01264_b200 import _native as N

    idx = torch.as_tensor(memory.sample_indices(B, np.random.default_rng(7)), device="cuda")
    theta, opt, target = fresh()
    ref = DataParallelLearner(theta, opt, target, memory, B).shard_gradient(idx).clone()
    dp = DataParallelLearner(theta, opt, target, memory, B)
    big, rest = dp.buckets()
    assert big.numel() + sum(t.numel() for t in rest) == dp.grad.numel() == dnn.num_params(A)
    assert big.numel() == 512 * 3136 and rest[0].numel() == dnn.num_params(A) - 512 * 3136 - rest[1].numel()
    dp.grad.fill_(float("nan"))
    ev = torch.cuda.Event()
    ev.record()
    a = dp._args(idx)
    N.check(N.load().pq_learn_grad_ev(N.C.byref(a), dp.grad.data_ptr(), N.stream_ptr(),
                                      N.C.c_void_p(ev.cuda_event)), "learn_grad_ev")
    side = torch.cuda.Stream()
    side.wait_event(ev)
    with torch.cuda.stream(side):
        early = big.clone()
    torch.cuda.synchronize()
    assert torch.equal(early, ref[big.data_ptr() // 4 - dp.grad.data_ptr() // 4:][:big.numel()])
    assert torch.equal(dp.grad, ref)
