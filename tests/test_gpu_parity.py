"""Parity of the CUDA path with the CPU oracle (the reference's algorithm) on the same
seeded inputs, through the C ABI.

Bit-exact: replay index sampling (incl. the reference's golden vectors), the
frame-stack gather, prepopulation, epsilon-greedy draws and the env step.
Tolerance (bf16 tensor-core arithmetic vs the fp64 oracle, relative Frobenius):
Q-values <= 1e-2, TD targets <= 1e-2, fc2 gradient <= 2e-2, lower-layer gradients
<= 0.2 -- bf16 weight rounding flips ~0.1% of the ReLU masks and, at batch 32, that
moves the conv/fc1 gradients by ~7% exactly as 0.2% fp64 weight noise does
(tests/test_oracle.py::test_gradient_conditioning_under_weight_noise documents it).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2111_01264_b200 import nn as dnn  # noqa: E402
from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams, epsilon_at, \
    train_minibatch  # noqa: E402
from paper_2111_01264_b200.envs import FrameEnvSpec  # noqa: E402
from paper_2111_01264_b200.executor import DeviceRun, run  # noqa: E402
from paper_2111_01264_b200.replay import ReplayMemory, Transition, device_pcg, \
    sample_indices_device  # noqa: E402

from oracle import _lib as OK  # noqa: E402
from oracle import natcnn, replay as oreplay  # noqa: E402
from oracle.envs import SyntheticFrameEnv  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")
A = 18


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# --- replay sampling: bit-exact with numpy / the reference golden vectors -------------

def test_sample_indices_golden_vectors():
    g = np.load(os.path.join(GOLD, "pcg64.npz"))
    c = 0
    while f"int{c}_n" in g:
        n, B = (int(v) for v in g[f"int{c}_n"])
        st = torch.from_numpy(g[f"int{c}_s0"].view(np.int64).copy()).cuda()
        out = sample_indices_device(st, n, B)
        assert np.array_equal(out.cpu().numpy(), g[f"int{c}_out"]), c
        assert np.array_equal(st.cpu().numpy().view(np.uint64), g[f"int{c}_s1"]), c
        out2 = sample_indices_device(st, n, B // 2 + 1)
        assert np.array_equal(out2.cpu().numpy(), g[f"int{c}_out2"]), c
        assert np.array_equal(st.cpu().numpy().view(np.uint64), g[f"int{c}_s2"]), c
        c += 1


@pytest.mark.parametrize("n,count", [(1_000_000, 80_000), (50_000, 32), (7, 100_003),
                                     (3_000_000_000, 5000), (2, 1), (1, 10), (123457, 0)])
def test_sample_indices_match_numpy(n, count):
    for pre in (0, 1):
        rng = np.random.default_rng(np.random.SeedSequence(n + pre, spawn_key=(2, 0)))
        if pre:
            rng.integers(0, 3, size=1)  # leave a buffered uint32
        st = device_pcg(rng)
        out = sample_indices_device(st, n, count)
        expect = rng.integers(0, n, size=count)
        assert np.array_equal(out.cpu().numpy(), expect)
        from paper_2111_01264_b200.replay import pcg_state_from_generator
        assert np.array_equal(st.cpu().numpy().view(np.uint64), pcg_state_from_generator(rng))


def test_replay_memory_sample_advances_generator_like_reference():
    mem = ReplayMemory(16)
    env = SyntheticFrameEnv(5, episode_length=6)
    mem.prepopulate(env, 12, np.random.default_rng(3))
    ora = oreplay.ReplayMemory(16)
    ora.prepopulate(SyntheticFrameEnv(5, episode_length=6), 12, np.random.default_rng(3))
    r1, r2 = np.random.default_rng(9), np.random.default_rng(9)
    for _ in range(5):
        b = mem.sample(7, r1)
        idx = ora.sample_indices(7, r2)
        assert np.array_equal(b.idx.cpu().numpy(), idx)
    assert mem.version == ora.version == 12
    assert len(mem) == len(ora) == 12


# --- frame-stack gather: bit-exact ------------------------------------------------------

def test_gather_bit_exact_vs_oracle_host_push():
    env_a, env_b = SyntheticFrameEnv(11, episode_length=5), SyntheticFrameEnv(11, episode_length=5)
    mem, ora = ReplayMemory(40), oreplay.ReplayMemory(40)
    mem.prepopulate(env_a, 37, np.random.default_rng(2))   # host env -> push path
    ora.prepopulate(env_b, 37, np.random.default_rng(2))
    r1, r2 = np.random.default_rng(4), np.random.default_rng(4)
    b = mem.sample(64, r1)
    s, a, r, s2, term = b.gather()
    ref = oreplay.gather(ora.sample(64, r2))
    assert np.array_equal(s.cpu().numpy(), ref[0])
    assert np.array_equal(a.cpu().numpy(), ref[1])
    assert np.array_equal(r.cpu().numpy(), ref[2].astype(np.float32))
    assert np.array_equal(s2.cpu().numpy(), ref[3])
    assert np.array_equal(term.cpu().numpy().astype(bool), ref[4])


def test_fifo_eviction_and_snapshot():
    """pkg/tests/test_replay.py:44-65 on frame transitions."""
    env = SyntheticFrameEnv(1, episode_length=50)
    mem, ora = ReplayMemory(5), oreplay.ReplayMemory(5)
    rng = np.random.default_rng(0)
    state = env.reset(rng)
    trans = []
    for k in range(12):
        nxt, rew, done = env.step(k % 18, rng)
        trans.append(Transition(state, k % 18, rew, nxt, False))
        state = env.reset(rng) if done else nxt
    for t in trans:
        mem.push(t)
        ora.push(oreplay.Transition(t.state, t.action, t.reward, t.next_state, t.terminal))
    snap = mem.snapshot()
    assert [x.action for x in snap] == [t.action for t in trans[-5:]]
    for x, t in zip(snap, trans[-5:]):
        assert x.state.tobytes() == t.state.tobytes()
        assert x.next_state.tobytes() == t.next_state.tobytes()
    assert mem.version == 12 and len(mem) == 5


def test_device_prepopulate_bit_exact_vs_oracle():
    n = 700
    spec = FrameEnvSpec(key=77, episode_length=9, action_count=A)
    mem = ReplayMemory(1024)
    rng_dev = np.random.default_rng(np.random.SeedSequence(1, spawn_key=(4, 0)))
    mem.prepopulate(spec, n, rng_dev)
    ora = oreplay.ReplayMemory(1024)
    rng_ora = np.random.default_rng(np.random.SeedSequence(1, spawn_key=(4, 0)))
    ora.prepopulate(SyntheticFrameEnv(77, episode_length=9, action_count=A), n, rng_ora)
    assert rng_dev.bit_generator.state == rng_ora.bit_generator.state
    idx = torch.arange(n, device="cuda")
    s, a, r, s2, term = mem.gather(idx)
    ref = oreplay.gather([ora.item(i) for i in range(n)])
    assert np.array_equal(s.cpu().numpy(), ref[0])
    assert np.array_equal(s2.cpu().numpy(), ref[3])
    assert np.array_equal(a.cpu().numpy(), ref[1])
    assert np.array_equal(r.cpu().numpy(), ref[2].astype(np.float32))
    assert np.array_equal(term.cpu().numpy().astype(bool), ref[4])


# --- Q network vs the fp64 oracle ----------------------------------------------------------

def _nets(seed):
    spec = natcnn.nature_cnn(A)
    p = natcnn.init_params(spec, seed)
    flat = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p.weights, p.biases)])
    return spec, p, dnn.QNet.from_flat(flat, A)


def test_forward_vs_oracle():
    spec, p, net = _nets(11)
    x = np.random.default_rng(0).integers(0, 256, size=(32, 4, 84, 84), dtype=np.uint8)
    q = dnn.forward(net, x)
    assert rel(q, natcnn.forward(spec, p, x)) < 1e-2


def test_train_minibatch_vs_oracle():
    spec, p, theta = _nets(3)
    _, pt, target = _nets(4)
    env = SyntheticFrameEnv(21, episode_length=30, action_count=A)
    mem, ora = ReplayMemory(200), oreplay.ReplayMemory(200)
    mem.prepopulate(env, 150, np.random.default_rng(1))
    ora.prepopulate(SyntheticFrameEnv(21, episode_length=30, action_count=A), 150,
                    np.random.default_rng(1))
    batch = mem.sample(32, np.random.default_rng(5))
    obatch = oreplay.gather(ora.sample(32, np.random.default_rng(5)))
    # oracle with the GPU's fp32-stored rewards
    obatch = (obatch[0], obatch[1], obatch[2].astype(np.float32).astype(np.float64), obatch[3],
              obatch[4])
    op = natcnn.Opt.zeros(p)
    p2, o2, g_ref, t_ref = natcnn.train_minibatch(spec, p, op, obatch, pt, 0.99, return_grad=True)
    th2, op2, grad, qout, td = dnn._learn(theta, dnn.OptState.zeros(theta), target, mem.ring,
                                          mem.records, batch.idx, 32, gamma=0.99,
                                          want_grad=True, want_q=True)
    qo = natcnn.forward(spec, p, obatch[0])
    assert rel(qout[0].cpu().numpy(), qo) < 1e-2
    assert rel(td[:, 0].cpu().numpy(), t_ref) < 1e-2
    g = grad.cpu().numpy()
    gref = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(g_ref.weights, g_ref.biases)])
    offs = np.cumsum([0] + [o * i + o for o, i in dnn.layer_shapes(A)])
    for k in range(5):
        e = rel(g[offs[k]:offs[k + 1]], gref[offs[k]:offs[k + 1]])
        assert e < (2e-2 if k == 4 else 0.2), (k, e)
    new = th2.flat()
    pref = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p2.weights, p2.biases)])
    old = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p.weights, p.biases)])
    assert rel(new - old, pref - old) < 0.2
    assert np.abs(new - pref).max() < 1e-3


def test_train_minibatch_leaves_target_untouched():
    """pkg/tests/test_agent.py:212-218."""
    _, _, theta = _nets(3)
    _, _, target = _nets(4)
    snap = target.master.clone()
    env = FrameEnvSpec(key=5, episode_length=20, action_count=A)
    mem = ReplayMemory(100)
    mem.prepopulate(env, 60, np.random.default_rng(0))
    train_minibatch(theta, dnn.OptState.zeros(theta), mem.sample(32, np.random.default_rng(0)),
                    target, 0.99, dnn.OptConfig())
    assert torch.equal(snap, target.master)


def test_gradient_zero_at_loss_minimum():
    """pkg/tests/test_nn.py:153-162 (targets = the network's own Q)."""
    _, _, net = _nets(4)
    x = np.random.default_rng(1).integers(0, 256, size=(6, 4, 84, 84), dtype=np.uint8)
    a = np.random.default_rng(2).integers(A, size=6)
    q = dnn.forward(net, x)
    g = dnn.gradient(net, x, a, q[np.arange(6), a])
    assert all((w == 0).all() for w in g.weights + g.biases)


def test_rmsprop_hand_value_and_non_finite():
    """pkg/tests/test_nn.py:221-252 on the device optimizer kernel."""
    net = dnn.QNet.from_flat(np.zeros(dnn.num_params(A)), A)
    g = np.zeros(dnn.num_params(A))
    g[0] = 1.0
    p2, o2 = dnn.rmsprop_step(dnn.OptState.zeros(net), dnn.OptConfig(), net,
                              dnn.Parameters.from_flat(g, A))
    assert abs(float(o2.m[0]) - 0.05) < 1e-7 and abs(float(o2.v[0]) - 0.05) < 1e-7
    assert abs(float(p2.master[0]) - (-2.5e-4 / np.sqrt(0.0575))) < 1e-9
    g[1] = np.nan
    with pytest.raises(ValueError):
        dnn.rmsprop_step(dnn.OptState.zeros(net), dnn.OptConfig(), net,
                         dnn.Parameters.from_flat(g, A))


# --- acting: epsilon-greedy + env step bit-exact given the kernel's own Q rows --------------

def test_act_step_bit_exact_vs_oracle_env_and_select_action():
    hp = HyperParams(C=48, F=4, N=100, W=8, batch_size=32, total_steps=48, capacity=1000,
                     schedule=EpsilonSchedule(1.0, 0.1, 30), episode_length=4, seed=7)
    runner = DeviceRun(hp, use_graphs=False)
    runner.begin_epoch(0)
    from paper_2111_01264_b200.executor import ROLE_SAMPLER, derived_seed, rng_stream
    keys = [derived_seed(hp.seed, ROLE_SAMPLER, 1000 + j) for j in range(hp.W)]
    envs = [SyntheticFrameEnv(k, episode_length=4, action_count=A) for k in keys]
    rngs = [rng_stream(hp.seed, ROLE_SAMPLER, j) for j in range(hp.W)]
    states = [e.reset(r) for e, r in zip(envs, rngs)]
    qbuf = torch.empty((hp.W, A), dtype=torch.float32, device="cuda")
    from paper_2111_01264_b200 import _native as N
    for b in range(hp.C // hp.W):
        a = runner._act_args()
        a.q_out = qbuf.data_ptr()
        a.epoch_start = 0
        N.check(N.load().pq_act_step(N.C.byref(a), N.stream_ptr()), "act")
        torch.cuda.synchronize()
        q = qbuf.cpu().numpy().astype(np.float64)
        acts = runner.envs.actions.cpu().numpy()
        stack = runner.envs.stack.cpu().numpy()
        for j in range(hp.W):
            t_label = b * hp.W + j + 1
            st = OK.pcg_state_from_generator(rngs[j])
            act = OK.select_action(st, q[j], epsilon_at(t_label, hp.schedule))
            OK.pcg_state_to_generator(st, rngs[j])
            assert act == acts[j], (b, j)
            nxt, rew, done = envs[j].step(act, rngs[j])
            if done:
                nxt = envs[j].reset(rngs[j])
            dev_state = torch.zeros((4, 7056), dtype=torch.uint8, device="cuda")
            for c in range(4):
                if stack[j, c] >= 0:
                    dev_state[c] = runner.D.ring[int(stack[j, c])]
            assert dev_state.cpu().numpy().tobytes() == nxt.tobytes(), (b, j)
        assert np.array_equal(runner.envs.pcg_states(),
                              np.stack([OK.pcg_state_from_generator(r) for r in rngs]))


# --- executor: determinism and schedule --------------------------------------------------------

def test_run_is_deterministic_and_counts_transactions():
    hp = HyperParams(C=64, F=4, N=200, W=8, batch_size=32, total_steps=128, capacity=2000,
                     schedule=EpsilonSchedule(1.0, 0.1, 100), episode_length=7, seed=3)
    r1 = run(hp, graph_chunk=8)
    r2 = run(hp, use_graphs=False)
    assert r1.epoch_hashes == r2.epoch_hashes
    assert r1.to_csv_text() == r2.to_csv_text()
    c = r1.counters
    assert c["inference_batched_calls"] == 128 // 8
    assert c["acting_rows_from_target"] == 128
    assert c["train_calls"] == 128 // 4
    assert c["flush_pushes"] == 128 and c["dfreeze_violations"] == 0
    assert any(kind == "episode" for _, kind, _ in r1.events)


def test_host_env_run_matches_device_env_run():
    """End-to-end path (CPU envs + select_action, H2D frames / D2H Q-rows per block)
    reproduces the all-device executor bit-exactly."""
    hp = HyperParams(C=64, F=4, N=200, W=8, batch_size=32, total_steps=128, capacity=2000,
                     schedule=EpsilonSchedule(1.0, 0.1, 100), episode_length=7, seed=5)
    r_dev = run(hp, graph_chunk=8)
    r_host = run(hp, host_envs=True, graph_chunk=8)
    assert r_dev.epoch_hashes == r_host.epoch_hashes
    assert r_dev.to_csv_text() == r_host.to_csv_text()


def test_concurrent_run_equals_sequential_reference():
    """executor.run (two streams, graphs) reproduces the single-lane schedule
    bit-exactly (pkg/tests/test_executor.py:94-108 oracle equivalence)."""
    from paper_2111_01264_b200.executor import sequential_reference

    hp = HyperParams(C=64, F=4, N=200, W=8, batch_size=32, total_steps=192, capacity=2000,
                     schedule=EpsilonSchedule(1.0, 0.1, 100), episode_length=9, seed=11)
    assert run(hp, graph_chunk=8).to_csv_text() == sequential_reference(hp).to_csv_text()


def test_device_evaluation_matches_oracle_evaluate_policy():
    """evaluate_policy (envs.py:177-202): exactly N episodes on one rng stream, same
    returns as the oracle env driven by the same actions."""
    hp = HyperParams(C=64, F=4, N=200, W=8, batch_size=32, total_steps=128, capacity=2000,
                     eval_period=64, eval_episodes=5, eval_epsilon=0.3, episode_length=6,
                     seed=2)
    runner = DeviceRun(hp, use_graphs=False)
    from paper_2111_01264_b200.executor import ROLE_EVAL, derived_seed
    seed = derived_seed(hp.seed, ROLE_EVAL, 0)
    mean, std = runner.evaluate(runner.target, hp.eval_epsilon, hp.eval_episodes, seed)
    # oracle: the same env / stream; actions from the device Q rows via a single-state
    # forward of each visited state
    env = SyntheticFrameEnv(derived_seed(hp.seed, ROLE_EVAL, 1000), episode_length=6,
                            action_count=A)
    rng = np.random.default_rng(seed)
    rets = []
    for _ in range(hp.eval_episodes):
        state = env.reset(rng)
        total, done = 0.0, False
        while not done:
            q = dnn.forward(runner.target, state[None])[0]
            st = OK.pcg_state_from_generator(rng)
            act = OK.select_action(st, q, hp.eval_epsilon)
            OK.pcg_state_to_generator(st, rng)
            state, rew, done = env.step(act, rng)
            total += rew
        rets.append(total)
    assert (mean, std) == (float(np.mean(rets)), float(np.std(rets)))
    rec = run(hp, graph_chunk=8)
    assert [k for _, k, _ in rec.events].count("eval_mean") == 2
