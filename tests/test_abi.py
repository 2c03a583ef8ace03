"""CPU-side checks of the C-ABI library (no GPU compute): it loads, exports every entry
point include/paraq_b200.h declares, and its host-only functions match the oracle
bit-exactly (theta hash, host samplers = select_action + env.step)."""

import os
import re

import numpy as np
import pytest

from paper_2111_01264_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "paraq_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pq(?:64)?_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    for name in N.EXPORTS:
        assert name in syms, f"{name} bound in _native.py but not declared in the header"


def test_abi_constants():
    lib = N.load()
    assert lib.pq_abi_version() == 1
    assert lib.pq_num_params(18) == 1_693_362
    assert lib.pq_workspace_bytes(32, 18) > 0
    lay = N.workspace_layout(64, 18)
    for k in ("dY1p", "dY2p", "act1s2", "act1s2_t"):   # the shifted-conv buffers exist from batch 128
        assert lay.pop(k) == -1
    offs = list(lay.values())
    assert offs == sorted(offs) and offs[0] == 0
    big = N.workspace_layout(256, 18)
    assert big["dY1p"] > big["grad4"]


def test_theta_hash_matches_reference_definition():
    """nn.theta_hash (nn.py:223-229) over LE float64 bytes, layer order."""
    from oracle import natcnn

    rng = np.random.default_rng(0)
    p = natcnn.Params([rng.normal(size=(3, 4)), rng.normal(size=(2, 3))],
                      [rng.normal(size=3), rng.normal(size=2)])
    flat = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p.weights, p.biases)])
    h = N.load().pq_theta_hash_f64(flat.ctypes.data, flat.size)
    assert f"{h:016x}" == natcnn.theta_hash(p)
    f32 = flat.astype(np.float32)
    h32 = N.load().pq_theta_hash_f32(f32.ctypes.data, f32.size)
    flat32 = f32.astype(np.float64)
    assert h32 == N.load().pq_theta_hash_f64(flat32.ctypes.data, flat32.size)


def test_theta_hash_matches_live_reference(reference_paraq):
    from paraq.nn import init_network, theta_hash

    p = init_network([5, 7, 3], 21)
    flat = np.concatenate([np.r_[w.ravel(), b] for w, b in zip(p.weights, p.biases)])
    h = N.load().pq_theta_hash_f64(flat.ctypes.data, flat.size)
    assert f"{h:016x}" == theta_hash(p)


def test_host_samplers_bit_exact_vs_oracle_env_and_select_action():
    """csrc/host_env.cpp (the end-to-end path's CPU samplers) against the oracle frame
    env + the restated select_action, over episode ends and exploration."""
    from oracle import _lib as OK
    from oracle.envs import SyntheticFrameEnv

    from paper_2111_01264_b200.agent import EpsilonSchedule, epsilon_at
    from paper_2111_01264_b200.replay import pcg_state_from_generator

    W, A, L = 4, 18, 5
    fcap = 10_000
    lib = N.load()
    keys = [11, 22, 33, 44]
    envs = (N.PqHenv * W)()
    rngs = [np.random.default_rng(np.random.SeedSequence(9, spawn_key=(1, j))) for j in range(W)]
    for j in range(W):
        st = pcg_state_from_generator(rngs[j])
        for k in range(6):
            envs[j].pcg[k] = int(st[k])
        envs[j].key = keys[j]
        envs[j].episode = -1
    oenv = [SyntheticFrameEnv(k, episode_length=L, action_count=A) for k in keys]
    ostate = [e.reset(None) for e in oenv]
    frames = np.zeros((2 * W, 7056), dtype=np.uint8)
    stacks = np.zeros((W, 4), dtype=np.int32)
    seq = np.array([0], dtype=np.int64)
    lib.pq_henv_reset(N.C.addressof(envs), W, seq.ctypes.data, fcap, frames.ctypes.data,
                      stacks.ctypes.data)
    ring = {}
    for j in range(W):
        ring[int(stacks[j, 3])] = frames[j].copy()
    sched = EpsilonSchedule(1.0, 0.1, 40)
    nf = np.zeros(1, dtype=np.int32)
    recs = np.zeros((W, 8), dtype=np.int32)
    labels = np.zeros(2 * W, dtype=np.int64)
    rets = np.zeros(2 * W, dtype=np.float64)
    neps = np.zeros(1, dtype=np.int32)
    qrng = np.random.default_rng(3)
    for b in range(30):
        q = qrng.normal(size=(W, A)).astype(np.float32)
        q[:, 7] = q[:, 3] = q.max(axis=1) + 1  # ties -> lowest index
        first = int(seq[0])
        neps[0] = 0
        lib.pq_henv_step(N.C.addressof(envs), W, q.ctypes.data, A, L, 1 / 256, b * W + 1,
                         sched.start, sched.end, sched.anneal_steps, seq.ctypes.data, fcap,
                         frames.ctypes.data, nf.ctypes.data, stacks.ctypes.data,
                         recs.ctypes.data, labels.ctypes.data, rets.ctypes.data, neps.ctypes.data)
        for k in range(int(nf[0])):
            ring[(first + k) % fcap] = frames[k].copy()
        for j in range(W):
            st = OK.pcg_state_from_generator(rngs[j])
            a = OK.select_action(st, q[j].astype(np.float64), epsilon_at(b * W + j + 1, sched))
            OK.pcg_state_to_generator(st, rngs[j])
            assert a == recs[j, 5] & 0xFFFF
            nxt, rew, done = oenv[j].step(a, rngs[j])
            assert np.float64(rew).view(np.int64) == recs[j, 6:8].copy().view(np.int64)[0]
            assert bool(recs[j, 5] >> 16) == (done and not oenv[j].truncated)
            assert ring[int(recs[j, 4])].tobytes() == nxt[3].tobytes()
            if done:
                nxt = oenv[j].reset(rngs[j])
            dev_state = np.stack([ring[int(s)] if s >= 0 else np.zeros(7056, np.uint8)
                                  for s in stacks[j]])
            assert dev_state.tobytes() == nxt.tobytes()
            assert np.array_equal(np.array(list(envs[j].pcg), dtype=np.uint64),
                                  pcg_state_from_generator(rngs[j]))


def test_reference_nn_runs_on_plugin_module_interface(reference_paraq):
    """The plugin module exposes exactly the reference kernel-module contract
    (_kernels_numba.py:14-121), so paraq.nn can be pointed at it."""
    import paraq._kernels_numba as ref_k

    from paper_2111_01264_b200 import kernels as b200

    names = ["BACKEND_NAME", "affine_rows", "relu", "output_delta", "weight_grad", "bias_grad",
             "hidden_delta", "rmsprop_flat", "spin"]
    for nm in names:
        assert hasattr(ref_k, nm) and hasattr(b200, nm), nm
    assert b200.spin(1000) == ref_k.spin(1000)
