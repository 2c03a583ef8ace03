"""Executor-level parity with the UNMODIFIED reference executor (executor.py:341-637).

tests/golden/make_executor_golden.py ran `paraq.executor.run` / `sequential_reference`
over the synthetic frame env (its env_factory hook) with epsilon = 1 acting and
eval_epsilon = 1 evaluation, so the replay memory, the episode log and the evaluation
returns are independent of the network and pin the schedule: prepopulation, lockstep
t-labels, the blocking training events of the non-concurrent modes (flush, then one
minibatch; executor.py:436-440, :457-494), owner-major flushes (replay.py:82-93), ring
eviction (capacity 300 < 200 prepopulated + 192 acted), the trainer's index draws
(its final PCG64 state), the samplers' streams and the InferenceWorker counters of
every mode.  The device executor must reproduce all of it bit for bit: every stored
transition in insertion order (frame-stack digests, action, f64 reward, bootstrap
terminal), episodes, evaluations, events and counters.
"""

import hashlib
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams  # noqa: E402
from paper_2111_01264_b200.envs import FrameEnvSpec  # noqa: E402
from paper_2111_01264_b200.executor import DeviceRun, HostEnvRun  # noqa: E402

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "executor.npz"))
BASE = dict(C=64, F=4, N=200, batch_size=32, total_steps=192, capacity=300, seed=3,
            eval_period=64, eval_episodes=3, eval_epsilon=1.0, episode_length=7,
            terminal_p=0.05, schedule=EpsilonSchedule(1.0, 1.0, 1))
CASES = [("both_w8", "both", 8, "run"), ("concurrent_w8", "concurrent", 8, "run"),
         ("synchronized_w8", "synchronized", 8, "run"), ("standard_w1", "standard", 1, "run"),
         ("standard_w4_seq", "standard", 4, "seq"),
         ("synchronized_w16_seq", "synchronized", 16, "seq")]


def digest(a) -> int:
    b = np.ascontiguousarray(np.asarray(a, dtype=np.uint8)).tobytes()
    return int.from_bytes(hashlib.blake2b(b, digest_size=8).digest(), "little")


def check(runner, rec, name):
    g = {k.split("__", 1)[1]: GOLD[k] for k in GOLD.files if k.startswith(name + "__")}
    snap = runner.D.snapshot()
    assert runner.D.version == int(g["version"][0])
    assert np.array_equal(np.array([digest(t.state) for t in snap], dtype=np.uint64), g["s"])
    assert np.array_equal(np.array([digest(t.next_state) for t in snap], dtype=np.uint64), g["s2"])
    assert np.array_equal(np.array([t.action for t in snap]), g["a"])
    assert np.array_equal(np.array([t.reward for t in snap]), g["r"])  # f64, bit-exact
    assert np.array_equal(np.array([t.terminal for t in snap]), g["term"])
    assert np.array_equal(np.array(rec.episodes, dtype=np.float64).reshape(-1, 2), g["episodes"])
    assert np.array_equal(np.array(rec.evals, dtype=np.float64).reshape(-1, 3), g["evals"])
    events = [f"{s},{k},{v}" for s, k, v in rec.events if k != "theta_hash"]
    assert events == list(g["events"])
    assert {k: rec.counters[k] for k in g["counter_names"]} == \
        dict(zip(g["counter_names"], g["counter_values"].tolist()))
    assert np.array_equal(runner.trainer_pcg.cpu().numpy().view(np.uint64), g["trainer_pcg"])


def make_hp(mode, W):
    return HyperParams(**BASE, W=W).with_mode(mode)


@pytest.mark.parametrize("name,mode,W,entry", CASES)
def test_device_executor_matches_reference_executor(name, mode, W, entry):
    hp = make_hp(mode, W)
    runner = DeviceRun(hp, sequential=entry == "seq", use_graphs=entry == "run", graph_chunk=4)
    rec = runner.execute()
    check(runner, rec, name)
    assert np.array_equal(runner.envs.pcg_states(),
                          GOLD[name + "__sampler_pcg"])


@pytest.mark.parametrize("name,mode,W", [("both_w8", "both", 8),
                                         ("synchronized_w8", "synchronized", 8)])
def test_host_env_executor_matches_reference_executor(name, mode, W):
    """The end-to-end path (host samplers, H2D frames / D2H Q-rows per block)."""
    hp = make_hp(mode, W)
    runner = HostEnvRun(hp, graph_chunk=4)
    rec = runner.execute()
    check(runner, rec, name)


def test_env_factory_template_and_reference_signature():
    """run(hp, env_factory, sink) (executor.py:591): positional factory and sink; the
    factory's FrameEnvSpec configures the envs; anything else is rejected."""
    from paper_2111_01264_b200.executor import run

    hp = make_hp("both", 8)
    seen = []
    spec = FrameEnvSpec(key=0, episode_length=7, action_count=18, terminal_p=0.05)
    rec = run(hp, lambda: spec, lambda s, k, v: seen.append((s, k, v)))
    assert seen == rec.events and any(k == "episode" for _, k, _ in seen)
    with pytest.raises(ValueError):
        run(hp, lambda: object())


def test_async_evaluation_matches_streamed_evaluation():
    """The evaluation overlapped with the next epoch on its own stream (no sink) lands the
    same mean / std at the same place in the record as the synchronous one a streaming
    sink forces; 300 episodes also grow the eval env's episode log past its 256 entries
    and take many CUDA-graph chunks; greedy actions make it depend on the snapshot."""
    from paper_2111_01264_b200.executor import run

    hp = HyperParams(**{**BASE, "eval_episodes": 300, "eval_epsilon": 0.05, "episode_length": 3,
                        "total_steps": 256}, W=8).with_mode("both")
    streamed = []
    a = run(hp)
    b = run(hp, None, lambda s, k, v: streamed.append((s, k, v)))
    assert len(a.evals) == 4 and all(m is not None for _, m, _ in a.evals)
    assert a.evals == b.evals
    assert [e for e in a.events if e[1] != "theta_hash"] == [e for e in b.events if e[1] != "theta_hash"]
    assert streamed == b.events


def test_compact_frame_ring_wraps_like_host_allocation():
    """The ring holds ~(1 + reset rate) frames per transition: reset frames get slots in
    (step, sampler) order from the step's last CTA and the epoch's unused reservation is
    returned.  40 epochs wrap it many times (every prepopulated record evicted); the
    device samplers' memory must equal the host samplers' (their own compact allocation)
    transition for transition, and the runs must agree bit for bit."""
    hp = HyperParams(**{**BASE, "total_steps": 64 * 120, "eval_period": 0}, W=8).with_mode("both")
    dev = DeviceRun(hp, graph_chunk=4)
    a = dev.execute()
    host = HostEnvRun(hp, graph_chunk=4)
    b = host.execute()
    assert dev.D.frame_seq > 3 * dev.D.frame_capacity  # wrapped 3 times
    assert dev.D.frame_capacity < 1.5 * hp.capacity + 2 * 5 * hp.C + 2 * hp.W + 1024
    sa, sb = dev.D.snapshot(), host.D.snapshot()
    assert len(sa) == len(sb) == hp.capacity
    assert [digest(t.state) for t in sa] == [digest(t.state) for t in sb]
    assert [digest(t.next_state) for t in sa] == [digest(t.next_state) for t in sb]
    assert a.final_hash == b.final_hash and a.episodes == b.episodes
