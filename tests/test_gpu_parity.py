"""Parity of the CUDA path with the CPU oracle (the reference's algorithm) on the same
seeded inputs, through the C ABI.

Bit-exact: replay index sampling (incl. the reference's golden vectors), the
frame-stack gather (f64 rewards), prepopulation, epsilon-greedy draws and the env step.
Tolerance (bf16 tensor-core arithmetic vs the fp64 oracle with the device's storage
model, relative Frobenius): Q-values and TD targets <= 1e-3; stage outputs <= 1e-3;
every layer's gradient, the post-RMSProp update and the moments <= 1e-5 on identical
stage inputs (see the section comment below).
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
from oracle import blas, natcnn, replay as oreplay  # noqa: E402
import devtap  # noqa: E402
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
    assert np.array_equal(r.cpu().numpy(), ref[2])
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
    assert np.array_equal(r.cpu().numpy(), ref[2])
    assert np.array_equal(term.cpu().numpy().astype(bool), ref[4])


# --- Q network vs the fp64 oracle ----------------------------------------------------------
#
# Tolerances (north star: "rel 1e-3 for bf16"), relative Frobenius, on identical weights
# and minibatches.  The oracle (oracle/natcnn.py, the reference arithmetic in fp64) runs
# with the device's storage model (natcnn.Bf16Storage: bf16 W1..W4, bf16 conv
# activations and data gradients) so the comparison is well posed:
#   * chained (the oracle rounds its own values): Q-values of both networks and the TD
#     targets <= 1e-3 (measured ~2e-4);
#   * per stage, teacher-forced (each oracle stage reads the device's stored bf16 input
#     of that stage and its ReLU masks): every stored tensor equals the oracle's value
#     rounded to bf16 within 1e-3 (measured <= 6e-5), and every layer's weight and bias
#     gradient, the post-RMSProp parameter update and the moments within 1e-5, the
#     north star's fp32 bar (measured 2e-8 .. 2e-6 at batch 32 / 256 / 1024).  Chained gradients are not a well-posed comparison: a bf16
#     value within the accumulation error of a rounding boundary lands one ulp (2^-8)
#     away, and a ReLU pre-activation within it flips a whole unit's gradient
#     (natcnn.Bf16Storage docstring).

RTOL_BF16 = 1e-3   # north star: bf16 arithmetic
RTOL_STAGE = 1e-5  # teacher-forced gradients / update (fp32 accumulation on equal inputs)


def _nets(seed, bias_scale=0.0):
    spec = natcnn.nature_cnn(A)
    p = natcnn.init_params(spec, seed)
    if bias_scale:
        brng = np.random.default_rng(seed + 100)
        for b in p.biases:
            b[:] = brng.normal(scale=bias_scale, size=b.shape)
    flat = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p.weights, p.biases)])
    net = dnn.QNet.from_flat(flat, A)
    # the oracle runs on the device's fp32 master values
    dp = dnn.Parameters.from_flat(net.flat(), A)
    return spec, natcnn.Params(dp.weights, dp.biases), net


def _flat(p):
    return np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p.weights, p.biases)])


@pytest.mark.parametrize("W", [8, 128, 512])
def test_forward_vs_oracle_bf16_faithful(W):
    """Batched acting inference (configs[2] widths) vs the oracle forward."""
    spec, p, net = _nets(11, bias_scale=0.05)
    x = np.random.default_rng(W).integers(0, 256, size=(W, 4, 84, 84), dtype=np.uint8)
    q = dnn.forward(net, x)
    ref = natcnn.forward(spec, p, x, K=blas, store=natcnn.Bf16Storage())
    e = rel(q, ref)
    print(f"forward W={W}: rel {e:.2e}")
    assert e < RTOL_BF16


def _learner_case(B, seed=3, huber=None):
    spec, p, theta = _nets(seed, bias_scale=0.05)
    _, pt, target = _nets(seed + 1, bias_scale=0.05)
    n = max(2 * B, 300)
    env = FrameEnvSpec(key=21 + B, episode_length=30, action_count=A)
    mem = ReplayMemory(n)
    mem.prepopulate(env, n, np.random.default_rng(1))
    ora = oreplay.ReplayMemory(n)
    ora.prepopulate(SyntheticFrameEnv(21 + B, episode_length=30, action_count=A), n,
                    np.random.default_rng(1))
    batch = mem.sample(B, np.random.default_rng(5))
    obatch = oreplay.gather(ora.sample(B, np.random.default_rng(5)))
    opt = dnn.OptState.zeros(theta)
    g = torch.Generator(device="cuda").manual_seed(B)
    opt.m.copy_(torch.randn(opt.m.shape, device="cuda", generator=g) * 1e-3)
    opt.v.copy_(opt.m * opt.m + torch.rand(opt.v.shape, device="cuda", generator=g) * 1e-4)
    m0 = dnn.Parameters.from_flat(opt.m.cpu().numpy().astype(np.float64), A)
    v0 = dnn.Parameters.from_flat(opt.v.cpu().numpy().astype(np.float64), A)
    oopt = natcnn.Opt(m0.weights, m0.biases, v0.weights, v0.biases)
    th2, op2, grad, qout, td = dnn._learn(theta, opt, target, mem.ring, mem.records, batch.idx,
                                          B, gamma=0.99, want_grad=True, want_q=True,
                                          huber=huber)
    taps = devtap.learner_taps(B, A)
    return dict(spec=spec, p=p, pt=pt, theta=theta, obatch=obatch, oopt=oopt, th2=th2,
                op2=op2, grad=grad.cpu().numpy().astype(np.float64),
                qout=qout.cpu().numpy().astype(np.float64),
                td=td.cpu().numpy().astype(np.float64), taps=taps)


def _forced_stores(taps, B):
    """Teacher-forced storage models from the device taps.  The device's data gradients
    are those of the summed loss (agent.py:103-104 feeds the optimizer n x the mean
    gradient, and the device never divides); the oracle's chain is nn.gradient's mean
    loss, so they enter scaled by 1/n (exact: B is a power of two)."""
    on = natcnn.Bf16Storage(masks=[None, None, None, taps["h1"] > 0, None], acts=taps["online"],
                            deltas={k: v / B for k, v in taps["deltas"].items()})
    return on, natcnn.Bf16Storage(acts=taps["target"])


@pytest.mark.parametrize("B", [32, 256, 512, 1024])
def test_learner_step_vs_oracle_bf16_faithful(B):
    """agent.train_minibatch (agent.py:84-105) on the GPU vs the fp64 oracle: batch 32
    runs the cp.async / fused small-batch schedule, 256 and 1024 the TMA and
    shifted-descriptor kernels, 512 also the split-partial block head (k_head_block_split)."""
    c = _learner_case(B)
    spec, p, pt, obatch, taps = c["spec"], c["p"], c["pt"], c["obatch"], c["taps"]
    s, a, r, s2, term = obatch
    # -- chained: the oracle rounds its own values where the device stores bf16
    q_on = natcnn.forward(spec, p, s, K=blas, store=natcnn.Bf16Storage())
    q_tg = natcnn.forward(spec, pt, s2, K=blas, store=natcnn.Bf16Storage())
    t_ref = natcnn.td_targets(spec, pt, r, s2, term, 0.99, K=blas, store=natcnn.Bf16Storage())
    errs = {"Q": rel(c["qout"][0], q_on), "Q_target": rel(c["qout"][1], q_tg),
            "td_target": rel(c["td"][:, 0], t_ref)}
    # -- teacher-forced: every stage on the device's stored inputs and masks
    st_on, st_tg = _forced_stores(taps, B)
    p2, o2, g_ref, t_forced = natcnn.train_minibatch(spec, p, c["oopt"], obatch, pt, 0.99,
                                                     return_grad=True, K=blas, store=st_on,
                                                     target_store=st_tg)
    errs["td_target_forced"] = rel(c["td"][:, 0], t_forced)
    for key, val in sorted(st_on.seen.items()):
        if key[0] == "act":
            dev, mine = taps["online"][key[1]], val
        else:  # the device's data gradients carry the summed-loss scale (x n)
            dev, mine = taps["deltas"][key[1]], val * B
        errs[f"stage_{key[0]}{key[1]}"] = rel(dev.reshape(-1), natcnn.bf16_round(mine).reshape(-1))
    for key, val in sorted(st_tg.seen.items()):
        errs[f"stage_target_{key[0]}{key[1]}"] = rel(taps["target"][key[1]].reshape(-1),
                                                     natcnn.bf16_round(val).reshape(-1))
    offs = np.cumsum([0] + [o * i + o for o, i in dnn.layer_shapes(A)])
    for k, (o, i) in enumerate(dnn.layer_shapes(A)):
        gw = c["grad"][offs[k]:offs[k] + o * i]
        gb = c["grad"][offs[k] + o * i:offs[k + 1]]
        errs[f"grad_w{k + 1}"] = rel(gw, g_ref.weights[k].ravel())
        errs[f"grad_b{k + 1}"] = rel(gb, g_ref.biases[k])
    old = _flat(p)
    errs["dtheta"] = rel(c["th2"].flat() - old, _flat(p2) - old)
    errs["m"] = rel(c["op2"].m.cpu().numpy(), _flat(natcnn.Params(o2.m_weights, o2.m_biases)))
    errs["v"] = rel(c["op2"].v.cpu().numpy(), _flat(natcnn.Params(o2.v_weights, o2.v_biases)))
    print(f"learner B={B}: " + ", ".join(f"{k} {v:.1e}" for k, v in errs.items()))
    for k, v in errs.items():
        bound = RTOL_STAGE if k.startswith(("grad", "dtheta", "m", "v", "td_target_")) \
            else RTOL_BF16
        assert v < bound, (k, v, bound)


@pytest.mark.parametrize("huber", [0.5, 2.0])
def test_learner_step_huber_vs_oracle(huber):
    """Opt-in Huber TD loss (north star): dL/dq clipped to [-delta, delta]; the default
    (huber unset) is the reference's half-squared loss (nn.py:140-144)."""
    B = 32
    c = _learner_case(B, seed=5, huber=huber)
    taps = c["taps"]
    d_dev = c["td"][:, 1]
    assert np.all(np.abs(d_dev) <= huber + 1e-7)
    assert np.any(np.abs(d_dev) == np.float32(huber)), "no clipped sample: pick a smaller delta"
    st_on, st_tg = _forced_stores(taps, B)
    p2, _, g_ref, _ = natcnn.train_minibatch(c["spec"], c["p"], c["oopt"], c["obatch"], c["pt"],
                                             0.99, return_grad=True, K=blas, store=st_on,
                                             target_store=st_tg, huber=huber)
    assert rel(c["grad"], _flat(g_ref)) < RTOL_STAGE
    old = _flat(c["p"])
    assert rel(c["th2"].flat() - old, _flat(p2) - old) < RTOL_STAGE


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
                     schedule=EpsilonSchedule(1.0, 0.1, 30), episode_length=4, seed=7, eval_period=0)
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
                     schedule=EpsilonSchedule(1.0, 0.1, 100), episode_length=7, seed=3, eval_period=0)
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
                     schedule=EpsilonSchedule(1.0, 0.1, 100), episode_length=7, seed=5, eval_period=0)
    r_dev = run(hp, graph_chunk=8)
    r_host = run(hp, host_envs=True, graph_chunk=8)
    assert r_dev.epoch_hashes == r_host.epoch_hashes
    assert r_dev.to_csv_text() == r_host.to_csv_text()


def test_concurrent_run_equals_sequential_reference():
    """executor.run (two streams, graphs) reproduces the single-lane schedule
    bit-exactly (pkg/tests/test_executor.py:94-108 oracle equivalence)."""
    from paper_2111_01264_b200.executor import sequential_reference

    hp = HyperParams(C=64, F=4, N=200, W=8, batch_size=32, total_steps=192, capacity=2000,
                     schedule=EpsilonSchedule(1.0, 0.1, 100), episode_length=9, seed=11, eval_period=0)
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


def test_gather_engines_bit_identical():
    """pq_replay_gather's TMA bulk-copy engine and the 16-byte-load engine agree byte for
    byte, incl. masked slots, a batch that is not a multiple of the persistent grid, and
    f64 rewards."""
    from paper_2111_01264_b200 import _native as N

    mem = ReplayMemory(3000)
    mem.prepopulate(FrameEnvSpec(key=8, episode_length=5, terminal_p=0.1), 2500, np.random.default_rng(3))
    B = 1237
    idx = torch.as_tensor(np.random.default_rng(4).integers(0, 2500, B), device="cuda")
    outs = []
    for fn in (N.load().pq_replay_gather_tma, N.load().pq_replay_gather_ldg):
        s = torch.full((B, 4, 84, 84), 7, dtype=torch.uint8, device="cuda")
        s2 = torch.full_like(s, 9)
        a = torch.empty(B, dtype=torch.int32, device="cuda")
        r = torch.empty(B, dtype=torch.float64, device="cuda")
        t = torch.empty(B, dtype=torch.uint8, device="cuda")
        N.check(fn(mem.ring.data_ptr(), mem.records.data_ptr(), idx.data_ptr(), B, s.data_ptr(), s2.data_ptr(),
                   a.data_ptr(), r.data_ptr(), t.data_ptr(), N.stream_ptr()), "gather")
        outs.append([x.cpu().numpy() for x in (s, s2, a, r, t)])
    for x, y in zip(*outs):
        assert np.array_equal(x, y)
    assert (outs[0][0] == 0).any()  # masked history frames present
