"""The reference's own agent / replay tests (pkg/tests/test_agent.py:124-218,
pkg/tests/test_replay.py:44-149), run against this package's modules with frame-stack
transitions in place of the reference's small float vectors.  Same assertions, same
API calls (list-of-Transition batches, ReplayMemory.sample returning Transitions,
flush over SampleBuffers, td_targets / train_minibatch on those batches)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.envs import SyntheticFrameEnv  # noqa: E402
from paper_2111_01264_b200 import nn as dnn  # noqa: E402
from paper_2111_01264_b200.agent import target_update, td_targets, train_minibatch  # noqa: E402
from paper_2111_01264_b200.nn import OptConfig, OptState, forward, init_network, \
    network_sizes, theta_hash  # noqa: E402
from paper_2111_01264_b200.replay import ReplayMemory, SampleBuffer, Transition  # noqa: E402

CHI2_CRIT_DF3_P001 = 16.266


def frame_transitions(n, key=1, terminal_every=None, seed=0):
    """n consecutive env transitions (episodes chained like the samplers do)."""
    env = SyntheticFrameEnv(key, episode_length=terminal_every or 10_000)
    rng = np.random.default_rng(seed)
    s = env.reset(rng)
    out = []
    for k in range(n):
        a = int(rng.integers(18))
        s2, r, done = env.step(a, rng)
        out.append(Transition(s, a, r, s2, done and not env.truncated))
        s = env.reset(rng) if done else s2
    return out


def tagged(ts, tags):
    """The same transitions with the reward replaced by a tag (test_replay.make_transition)."""
    return [Transition(t.state, t.action, float(g), t.next_state, t.terminal) for t, g in zip(ts, tags)]


# --- agent: targets (test_agent.py:124-158) --------------------------------------------

def test_terminal_target_is_reward_alone():
    net = init_network(network_sizes(), 0)
    t = frame_transitions(1)[0]
    batch = [Transition(t.state, t.action, 1.0, t.next_state, True)]
    assert td_targets(batch, net, 0.99).tolist() == [1.0]


def test_gamma_zero_targets_equal_rewards():
    net = init_network(network_sizes(), 0)
    ts = tagged(frame_transitions(2), [0.25, -0.5])
    assert td_targets(ts, net, 0.0).tolist() == [0.25, -0.5]


def test_td_targets_hand_computed_bootstrap():
    net = init_network(network_sizes(), 3)
    ts = tagged(frame_transitions(3), [0.5, 0.1, -0.2])
    q = forward(net, np.stack([t.next_state for t in ts])).astype(np.float64)
    expect = np.array([t.reward for t in ts]) + 0.9 * q.max(axis=1)
    assert np.array_equal(td_targets(ts, net, 0.9), expect)
    with pytest.raises(ValueError):
        td_targets([], net, 0.99)


# --- agent: train_minibatch (test_agent.py:164-218) ------------------------------------

def test_training_on_satisfied_targets_is_identity():
    theta = init_network(network_sizes(), 0)
    ts = frame_transitions(2)
    q = forward(theta, np.stack([t.state for t in ts]))
    batch = [Transition(t.state, t.action, float(q[i, t.action]), t.next_state, True)
             for i, t in enumerate(ts)]
    theta2, _ = train_minibatch(theta, OptState.zeros(theta), batch, target_update(theta), 0.99,
                                OptConfig())
    assert theta_hash(theta2) == theta_hash(theta)


def test_train_minibatch_is_deterministic():
    theta = init_network(network_sizes(), 1)
    target = target_update(theta)
    ts = frame_transitions(8, seed=3)
    a, _ = train_minibatch(theta, OptState.zeros(theta), ts, target, 0.99, OptConfig())
    b, _ = train_minibatch(theta, OptState.zeros(theta), ts, target, 0.99, OptConfig())
    assert theta_hash(a) == theta_hash(b)


def test_train_minibatch_decreases_loss_with_default_lr():
    theta = init_network(network_sizes(), 2)
    target = target_update(theta)
    ts = frame_transitions(16, seed=4)
    states = np.stack([t.state for t in ts])
    actions = np.asarray([t.action for t in ts])

    def loss(params):
        err = td_targets(ts, target, 0.99) - forward(params, states)[np.arange(16), actions]
        return float(np.mean(0.5 * err ** 2))

    before = loss(theta)
    theta2, _ = train_minibatch(theta, OptState.zeros(theta), ts, target, 0.99, OptConfig())
    assert loss(theta2) < before


def test_train_minibatch_leaves_target_untouched():
    theta = init_network(network_sizes(), 4)
    target = target_update(theta)
    snap = theta_hash(target)
    train_minibatch(theta, OptState.zeros(theta), frame_transitions(1), target, 0.99, OptConfig())
    assert theta_hash(target) == snap


# --- replay (test_replay.py:44-149) ---------------------------------------------------

def test_push_fifo_eviction():
    mem = ReplayMemory(2)
    for t in tagged(frame_transitions(3), (1.0, 2.0, 3.0)):
        mem.push(t)
    assert [t.reward for t in mem.snapshot()] == [2.0, 3.0]


def test_push_counts_and_version():
    mem = ReplayMemory(4)
    assert len(mem) == 0
    ts = frame_transitions(11)
    mem.push(ts[0])
    assert len(mem) == 1
    for t in ts[1:]:
        mem.push(t)
    assert len(mem) == 4 and mem.version == 11


def test_sample_single_item_gives_copies():
    mem = ReplayMemory(8)
    mem.push(tagged(frame_transitions(1), [9.0])[0])
    batch = mem.sample(32, np.random.default_rng(0))
    assert len(batch) == 32
    assert all(t.reward == 9.0 for t in batch)


def test_sample_is_deterministic_given_seed():
    mem = ReplayMemory(16)
    for t in tagged(frame_transitions(10), range(10)):
        mem.push(t)
    a = [t.reward for t in mem.sample(20, np.random.default_rng(42))]
    b = [t.reward for t in mem.sample(20, np.random.default_rng(42))]
    assert a == b


def test_sample_empty_memory_is_an_error():
    with pytest.raises(ValueError):
        ReplayMemory(4).sample(1, np.random.default_rng(0))


def test_sample_uniformity_binomial_bound():
    mem = ReplayMemory(4)
    for t in tagged(frame_transitions(4), range(4)):
        mem.push(t)
    draws = [t.reward for t in mem.sample(10_000, np.random.default_rng(7))]
    counts = np.bincount(np.asarray(draws, dtype=int), minlength=4)
    sigma = np.sqrt(10_000 * 0.25 * 0.75)
    assert (np.abs(counts - 2500) < 5 * sigma).all()
    assert float(((counts - 2500.0) ** 2 / 2500.0).sum()) < CHI2_CRIT_DF3_P001


def test_prepopulate_deterministic_and_resets_episodes():
    def fill(seed):
        mem = ReplayMemory(600)
        mem.prepopulate(SyntheticFrameEnv(5, episode_length=3), 500, np.random.default_rng(seed))
        return mem

    a, b = fill(5), fill(5)
    assert len(a) == 500
    for ta, tb in zip(a.snapshot(), b.snapshot()):
        assert ta.state.tobytes() == tb.state.tobytes()
        assert ta.action == tb.action and ta.reward == tb.reward and ta.terminal == tb.terminal
    with pytest.raises(ValueError):
        ReplayMemory(3).prepopulate(SyntheticFrameEnv(5), 4, np.random.default_rng(0))
    z = ReplayMemory(10)
    z.prepopulate(SyntheticFrameEnv(5), 0, np.random.default_rng(0))
    assert len(z) == 0 and z.version == 0


def test_flush_owner_order_then_chronological_and_idempotent():
    ts = tagged(frame_transitions(3), (1.0, 2.0, 3.0))
    mem = ReplayMemory(10)
    b0, b1 = SampleBuffer(0), SampleBuffer(1)
    b0.append(ts[0])
    b0.append(ts[1])
    b1.append(ts[2])
    assert mem.flush([b1, b0]) == 3  # argument order must not matter
    assert [t.reward for t in mem.snapshot()] == [1.0, 2.0, 3.0]
    assert len(b0) == 0 and len(b1) == 0
    v = mem.version
    assert mem.flush([b0, b1]) == 0 and mem.version == v


def test_batch_is_a_list_of_transitions():
    mem = ReplayMemory(64)
    mem.prepopulate(SyntheticFrameEnv(9, episode_length=5), 50, np.random.default_rng(1))
    batch = mem.sample(16, np.random.default_rng(2))
    s, a, r, s2, term = batch.gather()
    items = list(batch)
    assert len(items) == 16 and isinstance(items[0], Transition)
    assert np.array_equal(np.stack([t.state for t in items]), s.cpu().numpy())
    assert np.array_equal(np.stack([t.next_state for t in items]), s2.cpu().numpy())
    assert [t.action for t in items] == a.cpu().numpy().tolist()
    assert batch[3].reward == float(r[3])
    # a list of Transitions trains exactly like the device batch it came from
    theta, target = init_network(network_sizes(), 6), init_network(network_sizes(), 7)
    t1, _ = train_minibatch(theta, OptState.zeros(theta), batch, target, 0.99, OptConfig())
    t2, _ = train_minibatch(theta, OptState.zeros(theta), items, target, 0.99, OptConfig())
    assert torch.equal(t1.master, t2.master)
    assert dnn.num_params() == t1.master.numel()
