"""Pins the CPU oracle against the reference's own outputs (tests/golden/*.npz made by
tests/golden/make_golden.py from the unmodified reference) and against the
reference's known-answer tests (pkg/tests/test_nn.py, test_agent.py)."""

import math
import os

import numpy as np
import pytest

from oracle import _lib as K
from oracle import natcnn, replay as oreplay
from oracle.envs import SyntheticFrameEnv, make_frame

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


# --- kernels: bit-exact with the reference numba backend --------------------------

@pytest.mark.parametrize("case", [0, 1, 2])
def test_kernels_bit_exact_vs_reference_golden(case):
    g = gold("kernels.npz")
    c = str(case)
    w, b, x = g[f"aff{c}_w"], g[f"aff{c}_b"], g[f"aff{c}_x"]
    assert K.affine_rows(w, b, x).tobytes() == g[f"aff{c}_out"].tobytes()
    assert K.relu(x).tobytes() == g[f"relu{c}_out"].tobytes()
    assert K.output_delta(g[f"od{c}_q"], g[f"od{c}_a"], g[f"od{c}_t"]).tobytes() == \
        g[f"od{c}_out"].tobytes()
    delta, acts = g[f"wg{c}_delta"], g[f"wg{c}_acts"]
    assert K.weight_grad(delta, acts).tobytes() == g[f"wg{c}_out"].tobytes()
    assert K.bias_grad(delta).tobytes() == g[f"bg{c}_out"].tobytes()
    assert K.hidden_delta(delta, g[f"hd{c}_w"], g[f"hd{c}_pre"]).tobytes() == \
        g[f"hd{c}_out"].tobytes()
    p, gg, m, v = g[f"rms{c}_in"]
    out = np.stack(K.rmsprop_flat(p, gg, m, v, 2.5e-4, 0.95, 0.01))
    assert out.tobytes() == g[f"rms{c}_out"].tobytes()


def test_kernels_bit_exact_multithreaded():
    g = gold("kernels.npz")
    K.set_threads(4)
    try:
        w, x = g["aff1_w"], g["aff1_x"]
        big_x = np.tile(x, (400, 1))
        single = None
        K.set_threads(1)
        single = K.affine_rows(w, g["aff1_b"], big_x)
        K.set_threads(4)
        assert K.affine_rows(w, g["aff1_b"], big_x).tobytes() == single.tobytes()
        delta = np.tile(g["wg1_delta"], (400, 1))
        acts = np.tile(g["wg1_acts"], (400, 1))
        K.set_threads(1)
        s = K.weight_grad(delta, acts)
        K.set_threads(4)
        assert K.weight_grad(delta, acts).tobytes() == s.tobytes()
    finally:
        K.set_threads(1)


# --- PCG64 / Lemire / select_action restatement -------------------------------------

def test_pcg64_integers_bit_exact_vs_numpy_golden():
    g = gold("pcg64.npz")
    c = 0
    while f"int{c}_n" in g:
        n, B = (int(v) for v in g[f"int{c}_n"])
        s = g[f"int{c}_s0"].copy()
        assert np.array_equal(K.pcg64_integers(s, n, B), g[f"int{c}_out"]), c
        assert np.array_equal(s, g[f"int{c}_s1"]), c
        assert np.array_equal(K.pcg64_integers(s, n, B // 2 + 1), g[f"int{c}_out2"]), c
        assert np.array_equal(s, g[f"int{c}_s2"]), c
        c += 1
    assert c >= 9


def test_pcg64_random_and_select_action_bit_exact():
    g = gold("pcg64.npz")
    s = g["rand_s0"].copy()
    vals = np.array([K.pcg64_random(s) for _ in range(100)])
    assert vals.tobytes() == g["rand_out"].tobytes()
    assert np.array_equal(s, g["rand_s1"])
    s = g["sel_s0"].copy()
    acts = [K.select_action(s, g["sel_q"][i], float(g["sel_eps"][i])) for i in range(500)]
    assert np.array_equal(acts, g["sel_out"])
    assert np.array_equal(s, g["sel_s1"])


def test_pcg_state_roundtrip_through_numpy_generator():
    rng = np.random.default_rng(77)
    rng.integers(0, 9, size=3)
    st = K.pcg_state_from_generator(rng)
    expect = rng.integers(0, 1000, size=50)
    K.pcg_state_to_generator(st, rng)
    assert np.array_equal(rng.integers(0, 1000, size=50), expect)


# --- composition: the oracle's MLP path reproduces reference nn / agent bit-exactly --

def _mlp_params(g, prefix, n):
    return natcnn.Params([g[f"{prefix}_w{k}"] for k in range(n)],
                         [g[f"{prefix}_b{k}"] for k in range(n)])


def test_mlp_forward_gradient_train_bit_exact_vs_reference_golden():
    g = gold("mlp.npz")
    spec = natcnn.mlp([6, 9, 5, 4])
    theta = _mlp_params(g, "theta", 3)
    target = _mlp_params(g, "target", 3)
    assert natcnn.forward(spec, theta, g["states"]).tobytes() == g["q"].tobytes()
    gr = natcnn.gradient(spec, theta, g["states"], g["actions"], g["targets"])
    for k in range(3):
        assert gr.weights[k].tobytes() == g[f"grad_w{k}"].tobytes()
        assert gr.biases[k].tobytes() == g[f"grad_b{k}"].tobytes()
    batch = (g["states"], g["actions"], g["rewards"], g["next_states"], g["terminals"])
    opt = natcnn.Opt.zeros(theta)
    p1, o1 = natcnn.train_minibatch(spec, theta, opt, batch, target, 0.99)
    p2, o2 = natcnn.train_minibatch(spec, p1, o1, batch, target, 0.99)
    for k in range(3):
        assert p2.weights[k].tobytes() == g[f"p2_w{k}"].tobytes()
        assert p2.biases[k].tobytes() == g[f"p2_b{k}"].tobytes()
        assert o2.m_weights[k].tobytes() == g[f"m2_w{k}"].tobytes()
        assert o2.v_weights[k].tobytes() == g[f"v2_w{k}"].tobytes()


def test_replay_restatement_matches_reference_golden():
    g = gold("replay.npz")
    mem = oreplay.ReplayMemory(37)
    rng = np.random.default_rng(np.random.SeedSequence(5, spawn_key=(2, 0)))
    bufs = {2: [], 0: [], 1: []}
    tag = 0
    for epoch in range(6):
        for step in range(5):
            for owner in (2, 0, 1):
                bufs[owner].append(oreplay.Transition(None, 0, float(tag), None, False))
                tag += 1
        mem.flush(bufs)
        idx = mem.sample_indices(16, rng)
        assert np.array_equal(idx, g["idx"][epoch])
        assert [mem.item(i).reward for i in idx] == list(g["tags"][epoch])
        assert len(mem) == g["length"][epoch]
        assert mem.version == g["version"][epoch]


# --- reference known-answer tests, restated on the oracle ----------------------------

def test_rmsprop_hand_value():
    """pkg/tests/test_nn.py:221-230 / test_acceptance.py:93-106."""
    p = natcnn.Params([np.array([[0.0]])], [np.array([0.0])])
    g = natcnn.Params([np.array([[1.0]])], [np.array([0.0])])
    p2, o2 = natcnn.rmsprop_step(natcnn.Opt.zeros(p), p, g)
    assert o2.m_weights[0][0, 0] == pytest.approx(0.05, abs=1e-12)
    assert o2.v_weights[0][0, 0] == pytest.approx(0.05, abs=1e-12)
    assert p2.weights[0][0, 0] == pytest.approx(-2.5e-4 / math.sqrt(0.0575), abs=1e-12)


def test_rmsprop_rejects_non_finite():
    """pkg/tests/test_nn.py:247-252."""
    p = natcnn.Params([np.zeros((2, 2))], [np.zeros(2)])
    g = natcnn.Params([np.array([[np.nan, 0.0], [0.0, 0.0]])], [np.zeros(2)])
    with pytest.raises(ValueError):
        natcnn.rmsprop_step(natcnn.Opt.zeros(p), p, g)


def test_hand_linear_gradient():
    """pkg/tests/test_nn.py:165-175."""
    spec = natcnn.mlp([2, 2])
    p = natcnn.Params([np.array([[0.5, -0.25], [0.1, 0.2]])], [np.array([0.05, -0.1])])
    g = natcnn.gradient(spec, p, np.array([[1.0, 2.0]]), np.array([0]), np.array([3.0]))
    np.testing.assert_allclose(g.weights[0], [[-2.95, -5.9], [0.0, 0.0]], atol=1e-15)


def test_td_targets_hand_values():
    """pkg/tests/test_agent.py:124-143: terminal -> r; gamma = 0 -> r; 0.5 + 0.9*0.6."""
    spec = natcnn.mlp([2, 2])
    p = natcnn.Params([np.array([[0.0, 0.6], [0.0, 0.1]])], [np.zeros(2)])
    nxt = np.array([[0.0, 1.0], [0.0, 1.0], [0.0, 1.0]])
    t = natcnn.td_targets(spec, p, [0.5, 0.5, 0.5], nxt, [False, True, False], 0.9)
    assert t[0] == pytest.approx(0.5 + 0.9 * 0.6)
    assert t[1] == 0.5
    t0 = natcnn.td_targets(spec, p, [0.25], nxt[:1], [False], 0.0)
    assert t0[0] == 0.25


# --- conv restatement: independent checks (torch conv2d in fp64, finite differences) -

def _small_cnn(actions=5):
    return natcnn.nature_cnn(actions=actions, frame=36)


def test_conv_forward_matches_torch_fp64():
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    spec = natcnn.nature_cnn(actions=18)
    p = natcnn.init_params(spec, 11)
    rng = np.random.default_rng(0)
    x = rng.integers(0, 256, size=(3, 4, 84, 84), dtype=np.uint8)
    q = natcnn.forward(spec, p, x)
    t = torch.from_numpy(x.astype(np.float64) / 255.0)
    w1 = torch.from_numpy(p.weights[0].reshape(32, 4, 8, 8))
    h = F.relu(F.conv2d(t, w1, torch.from_numpy(p.biases[0]), stride=4))
    w2 = torch.from_numpy(p.weights[1].reshape(64, 4, 4, 32)).permute(0, 3, 1, 2)
    h = F.relu(F.conv2d(h, w2, torch.from_numpy(p.biases[1]), stride=2))
    w3 = torch.from_numpy(p.weights[2].reshape(64, 3, 3, 64)).permute(0, 3, 1, 2)
    h = F.relu(F.conv2d(h, w3, torch.from_numpy(p.biases[2]), stride=1))
    h = h.permute(0, 2, 3, 1).reshape(3, -1)
    h = F.relu(h @ torch.from_numpy(p.weights[3]).T + torch.from_numpy(p.biases[3]))
    qt = h @ torch.from_numpy(p.weights[4]).T + torch.from_numpy(p.biases[4])
    np.testing.assert_allclose(q, qt.numpy(), rtol=1e-12, atol=1e-12)


def test_conv_gradient_matches_finite_differences():
    """The reference's own gradient oracle (pkg/tests/test_nn.py:29-53, :185-196)."""
    spec = _small_cnn()
    p = natcnn.init_params(spec, 5)
    rng = np.random.default_rng(1)
    x = rng.integers(0, 256, size=(3, 4, 36, 36), dtype=np.uint8)
    a = rng.integers(5, size=3)
    t = rng.normal(size=3)
    g = natcnn.gradient(spec, p, x, a, t)
    h = 1e-6
    worst = 0.0
    prng = np.random.default_rng(2)
    for arrs, garrs in ((p.weights, g.weights), (p.biases, g.biases)):
        for arr, garr in zip(arrs, garrs):
            flat, gflat = arr.reshape(-1), garr.reshape(-1)
            for i in prng.choice(flat.size, size=min(12, flat.size), replace=False):
                orig = flat[i]
                flat[i] = orig + h
                lp = natcnn.loss_value(spec, p, x, a, t)
                flat[i] = orig - h
                lm = natcnn.loss_value(spec, p, x, a, t)
                flat[i] = orig
                num = (lp - lm) / (2 * h)
                worst = max(worst, abs(num - gflat[i]) / max(abs(num), abs(gflat[i]), 1e-4))
    assert worst < 1e-5


def test_nature_cnn_param_count():
    assert natcnn.nature_cnn().n_params == 1_693_362


# --- synthetic frame env ---------------------------------------------------------------

def test_frame_env_deterministic_and_masked():
    e1 = SyntheticFrameEnv(key=123, episode_length=5)
    e2 = SyntheticFrameEnv(key=123, episode_length=5)
    r1, r2 = np.random.default_rng(0), np.random.default_rng(0)
    s1, s2 = e1.reset(r1), e2.reset(r2)
    assert s1.tobytes() == s2.tobytes()
    assert (s1[:3] == 0).all() and s1[3].any()
    for k in range(5):
        n1, rew1, d1 = e1.step(k % 18, r1)
        n2, rew2, d2 = e2.step(k % 18, r2)
        assert n1.tobytes() == n2.tobytes() and rew1 == rew2 and d1 == d2
        assert n1[:3].tobytes() == s1[1:].tobytes()
        s1 = n1
    assert d1 and e1.truncated
    assert not np.array_equal(make_frame(1, 0, 1, 3), make_frame(1, 0, 1, 4))


def test_reference_replay_accepts_frame_transitions(reference_paraq):
    """Live cross-check (here only): the reference ReplayMemory fed by the frame env
    yields the same sampled stacks as the oracle restatement."""
    from paraq.replay import ReplayMemory as RefMem

    env_a, env_b = SyntheticFrameEnv(9, episode_length=7), SyntheticFrameEnv(9, episode_length=7)
    ref, ora = RefMem(50), oreplay.ReplayMemory(50)
    ref.prepopulate(env_a, 40, np.random.default_rng(4))
    ora.prepopulate(env_b, 40, np.random.default_rng(4))
    ra, rb = np.random.default_rng(8), np.random.default_rng(8)
    bref = ref.sample(16, ra)
    bora = ora.sample(16, rb)
    for x, y in zip(bref, bora):
        assert x.state.tobytes() == y.state.tobytes()
        assert x.next_state.tobytes() == y.next_state.tobytes()
        assert (x.action, x.reward, x.terminal) == (y.action, y.reward, y.terminal)


def _cnn_case(B=4, seed=11):
    spec = natcnn.nature_cnn(18)
    p = natcnn.init_params(spec, seed)
    rng = np.random.default_rng(seed)
    for b in p.biases:
        b[:] = rng.normal(scale=0.05, size=b.shape)
    x = rng.integers(0, 256, size=(B, 4, 84, 84), dtype=np.uint8)
    a = rng.integers(18, size=B)
    t = rng.normal(size=B)
    return spec, p, x, a, t


def test_blas_kernel_module_matches_exact_module():
    """oracle/blas.py (the reference numpy backend, batched rows) agrees with the
    bit-exact kernels.c module within the reference's own inter-backend tolerance
    (pkg/tests/test_backend.py:59-63: rtol 1e-12 on Q, 1e-10 on gradients)."""
    from oracle import blas

    spec, p, x, a, t = _cnn_case()
    np.testing.assert_allclose(natcnn.forward(spec, p, x, K=blas), natcnn.forward(spec, p, x),
                               rtol=1e-12, atol=1e-14)
    g1 = natcnn.gradient(spec, p, x, a, t)
    g2 = natcnn.gradient(spec, p, x, a, t, K=blas)
    for u, v in zip(g1.weights + g1.biases, g2.weights + g2.biases):
        np.testing.assert_allclose(v, u, rtol=1e-10, atol=1e-15)


def test_col2im_fast_matches_col2im():
    L = natcnn.Layer("conv", 64, 4, 2)
    dp = np.random.default_rng(0).normal(size=(2 * 81, 4 * 4 * 32))
    np.testing.assert_allclose(natcnn.col2im_fast(dp, L, (20, 20, 32), 2),
                               natcnn.col2im(dp, L, (20, 20, 32), 2), rtol=1e-13, atol=1e-15)


def test_bf16_round_is_round_to_nearest_even():
    # bf16 keeps 8 significant bits: one ulp at 1.0 is 2^-7
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, 1.0 + 2 ** -7 + 2 ** -8, -3.14159,
                  0.0, 1e-30, 65504.0])
    r = natcnn.bf16_round(x)
    assert r[0] == 1.0
    assert r[1] == 1.0                    # half ulp above an even value: ties to even
    assert r[2] == 1.0 + 2 ** -7          # 0.75 ulp rounds up
    assert r[3] == 1.0 + 2 ** -6          # half ulp above an odd value: ties to even (up)
    assert abs(r[4] + 3.140625) < 1e-12 and r[5] == 0.0
    assert np.all(np.abs(r - x) <= np.abs(x) * 2 ** -8 + 1e-45)
    # bf16 values are fixed points
    assert np.array_equal(natcnn.bf16_round(r), r)


def test_bf16_storage_model_points():
    """The storage model rounds W1..W4 (not fc2), the conv activations (not h1 / Q)
    and the data gradients; with identity-valued taps it reproduces itself."""
    spec, p, x, a, t = _cnn_case(B=2)
    st = natcnn.Bf16Storage()
    rows, pres, acts = natcnn.forward_trace(spec, p, x, store=st)
    for k in range(3):
        assert np.array_equal(natcnn.bf16_round(acts[k + 1]), acts[k + 1])
    assert not np.array_equal(natcnn.bf16_round(acts[4]), acts[4])   # h1 stays fp64
    assert np.array_equal(natcnn.bf16_round(rows[3]), rows[3])       # fc1 reads bf16 act3
    g = natcnn.gradient(spec, p, x, a, t, store=st)
    # teacher forcing with the model's own rounded values is the identity
    st2 = natcnn.Bf16Storage(acts={k: natcnn.bf16_round(st.seen[("act", k)]) for k in range(3)},
                             deltas={k: natcnn.bf16_round(st.seen[("delta", k)])
                                     for k in range(4)})
    g2 = natcnn.gradient(spec, p, x, a, t, store=st2)
    for u, v in zip(g.weights + g.biases, g2.weights + g2.biases):
        np.testing.assert_array_equal(u, v)


def test_huber_loss_gradient():
    """Opt-in Huber TD loss: delta = inf is the reference's half-squared loss; a finite
    delta clips dL/dq, and matches finite differences of the Huber loss."""
    spec = _small_cnn()
    p = natcnn.init_params(spec, 5)
    rng = np.random.default_rng(1)
    x = rng.integers(0, 256, size=(3, 4, 36, 36), dtype=np.uint8)
    a = rng.integers(5, size=3)
    t = np.array([10.0, -10.0, 0.01])
    g_sq = natcnn.gradient(spec, p, x, a, t)
    g_inf = natcnn.gradient(spec, p, x, a, t, huber=np.inf)
    for u, v in zip(g_sq.weights, g_inf.weights):
        np.testing.assert_array_equal(u, v)
    delta = 0.5
    g = natcnn.gradient(spec, p, x, a, t, huber=delta)

    def huber_loss(pp):
        q = natcnn.forward(spec, pp, x)
        e = q[np.arange(3), a] - t
        ae = np.abs(e)
        return float(np.mean(np.where(ae <= delta, 0.5 * e * e, delta * (ae - 0.5 * delta))))

    h = 1e-6
    w = p.weights[4]
    for i in range(5):
        orig = w.flat[i]
        w.flat[i] = orig + h
        lp = huber_loss(p)
        w.flat[i] = orig - h
        lm = huber_loss(p)
        w.flat[i] = orig
        num = (lp - lm) / (2 * h)
        assert abs(num - g.weights[4].flat[i]) <= 1e-6 * max(1.0, abs(num))
