"""Generate the golden fixtures by running the UNMODIFIED reference (`paraq`).

Run here (the container that has /root/reference):

    python tests/golden/make_golden.py

Outputs (committed, small):
* kernels.npz -- inputs/outputs of every reference numba kernel
  (_kernels_numba.py:19-111) on seeded inputs, incl. zeros in delta
  (the weight_grad skip, :63) and non-positive pre-activations (:88).
* pcg64.npz   -- Generator.integers(0, n, B) (replay.py:65) and random() draws
  with the full PCG64 state before/after, chained calls (has_uint32 carry), and
  select_action sequences (agent.py:53-66).
* mlp.npz     -- reference nn.forward / nn.gradient / agent.train_minibatch on a
  seeded dense net (pins the oracle's composition of the kernels).
* replay.npz  -- a reference ReplayMemory push / flush / sample sequence.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ["PARAQ_BACKEND"] = "numba"
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from paraq import _kernels_numba as K  # noqa: E402
from paraq.agent import select_action, train_minibatch  # noqa: E402
from paraq.nn import OptConfig, OptState, forward, gradient, init_network  # noqa: E402
from paraq.replay import ReplayMemory, SampleBuffer, Transition  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1


def pcg_state(rng):
    st = rng.bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    return np.array([s >> 64, s & M64, inc >> 64, inc & M64, st["has_uint32"], st["uinteger"]],
                    dtype=np.uint64)


def kernels():
    rng = np.random.default_rng(20211101)
    out = {}
    for case, (n, o, d) in enumerate([(5, 7, 11), (32, 18, 64), (3, 4, 257)]):
        w = rng.normal(size=(o, d))
        b = rng.normal(size=o)
        x = rng.normal(size=(n, d))
        out[f"aff{case}_w"], out[f"aff{case}_b"], out[f"aff{case}_x"] = w, b, x
        out[f"aff{case}_out"] = K.affine_rows(w, b, x)
        out[f"relu{case}_out"] = K.relu(x)
        q = rng.normal(size=(n, o))
        a = rng.integers(o, size=n)
        t = rng.normal(size=n)
        out[f"od{case}_q"], out[f"od{case}_a"], out[f"od{case}_t"] = q, a, t
        out[f"od{case}_out"] = K.output_delta(q, a, t)
        delta = rng.normal(size=(n, o)) * (rng.random((n, o)) < 0.6)
        acts = rng.normal(size=(n, d))
        out[f"wg{case}_delta"], out[f"wg{case}_acts"] = delta, acts
        out[f"wg{case}_out"] = K.weight_grad(delta, acts)
        out[f"bg{case}_out"] = K.bias_grad(delta)
        pre = rng.normal(size=(n, d))
        pre[rng.random((n, d)) < 0.1] = 0.0
        out[f"hd{case}_w"], out[f"hd{case}_pre"] = w, pre
        out[f"hd{case}_out"] = K.hidden_delta(delta, w, pre)
        k = n * o
        p, g, m = rng.normal(size=k), rng.normal(size=k), rng.normal(size=k) * 0.1
        v = m * m + rng.random(k)
        out[f"rms{case}_in"] = np.stack([p, g, m, v])
        p2, m2, v2 = K.rmsprop_flat(p, g, m, v, 2.5e-4, 0.95, 0.01)
        out[f"rms{case}_out"] = np.stack([p2, m2, v2])
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def pcg64():
    out = {}
    cases = [(7, 50), (10_000, 333), (999_983, 1000), (1_000_000, 4096), (2**31 + 12345, 777),
             (18, 64), (1, 5), (2, 9), (3, 1)]
    for c, (n, B) in enumerate(cases):
        rng = np.random.default_rng(np.random.SeedSequence(c, spawn_key=(2, 0)))
        if c % 2:                      # odd cases start with a buffered uint32
            rng.integers(0, 5, size=1)
        out[f"int{c}_n"] = np.array([n, B], dtype=np.int64)
        out[f"int{c}_s0"] = pcg_state(rng)
        out[f"int{c}_out"] = rng.integers(0, n, size=B)
        out[f"int{c}_s1"] = pcg_state(rng)
        out[f"int{c}_out2"] = rng.integers(0, n, size=B // 2 + 1)   # chained call
        out[f"int{c}_s2"] = pcg_state(rng)
    rng = np.random.default_rng(12345)
    rng.integers(0, 3, size=1)
    out["rand_s0"] = pcg_state(rng)
    out["rand_out"] = rng.random(100)
    out["rand_s1"] = pcg_state(rng)
    # select_action discipline (agent.py:53-66): 1 draw greedy, 2 when exploring
    rng = np.random.default_rng(np.random.SeedSequence(0, spawn_key=(1, 3)))
    qrng = np.random.default_rng(99)
    q = qrng.normal(size=(500, 18))
    q[::7, 5] = q[::7, 2] = 10.0  # ties -> lowest index
    eps = qrng.random(500)
    out["sel_s0"] = pcg_state(rng)
    out["sel_q"], out["sel_eps"] = q, eps
    out["sel_out"] = np.array([select_action(q[i], float(eps[i]), rng) for i in range(500)])
    out["sel_s1"] = pcg_state(rng)
    np.savez_compressed(os.path.join(OUT, "pcg64.npz"), **out)


def mlp():
    out = {}
    sizes = [6, 9, 5, 4]
    theta = init_network(sizes, 7)
    target = init_network(sizes, 8)
    rng = np.random.default_rng(3)
    n = 12
    states = rng.normal(size=(n, 6))
    next_states = rng.normal(size=(n, 6))
    actions = rng.integers(4, size=n)
    rewards = rng.random(n)
    terminals = rng.random(n) < 0.3
    targets = rng.normal(size=n)
    for k, (w, b) in enumerate(zip(theta.weights, theta.biases)):
        out[f"theta_w{k}"], out[f"theta_b{k}"] = w, b
    for k, (w, b) in enumerate(zip(target.weights, target.biases)):
        out[f"target_w{k}"], out[f"target_b{k}"] = w, b
    out.update(states=states, next_states=next_states, actions=actions, rewards=rewards,
               terminals=terminals, targets=targets)
    out["q"] = forward(theta, states)
    g = gradient(theta, states, actions, targets)
    for k in range(len(sizes) - 1):
        out[f"grad_w{k}"], out[f"grad_b{k}"] = g.weights[k], g.biases[k]
    batch = [Transition(states[i], int(actions[i]), float(rewards[i]), next_states[i],
                        bool(terminals[i])) for i in range(n)]
    opt = OptState.zeros(theta)
    p1, o1 = train_minibatch(theta, opt, batch, target, 0.99, OptConfig())
    p2, o2 = train_minibatch(p1, o1, batch, target, 0.99, OptConfig())
    for k in range(len(sizes) - 1):
        out[f"p2_w{k}"], out[f"p2_b{k}"] = p2.weights[k], p2.biases[k]
        out[f"m2_w{k}"], out[f"v2_w{k}"] = o2.m_weights[k], o2.v_weights[k]
    np.savez_compressed(os.path.join(OUT, "mlp.npz"), **out)


def replay():
    """Frame-stacked transitions through the reference ReplayMemory: tags are stored
    as the reward so the fixture stays tiny; the index stream is what is pinned."""
    mem = ReplayMemory(37)
    rng = np.random.default_rng(np.random.SeedSequence(5, spawn_key=(2, 0)))
    bufs = [SampleBuffer(j) for j in (2, 0, 1)]
    log_tags, log_idx, log_len, log_ver = [], [], [], []
    tag = 0
    for epoch in range(6):
        for step in range(5):
            for buf in bufs:
                buf.append(Transition(np.zeros(1), 0, float(tag), np.zeros(1), False))
                tag += 1
        mem.flush(bufs)
        idx = rng.integers(0, len(mem), size=16)
        batch = [mem._items[i] for i in idx]
        log_idx.append(idx)
        log_tags.append([t.reward for t in batch])
        log_len.append(len(mem))
        log_ver.append(mem.version)
    np.savez_compressed(os.path.join(OUT, "replay.npz"), idx=np.array(log_idx),
                        tags=np.array(log_tags), length=np.array(log_len),
                        version=np.array(log_ver))


if __name__ == "__main__":
    kernels()
    pcg64()
    mlp()
    replay()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
