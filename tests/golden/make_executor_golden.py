"""Executor-level goldens: run the UNMODIFIED reference executor (`paraq.executor.run`
and `sequential_reference`, executor.py:341-637) over the synthetic 84x84 frame env
and record what the device executor must reproduce bit for bit.

Run here (the container that has /root/reference):

    python tests/golden/make_executor_golden.py

The reference executor is driven through its own env_factory hook (executor.py:346)
with oracle/envs.SyntheticFrameEnv envs whose states are flattened uint8 [28224]
vectors (its MLP forward takes 2-D rows, nn.py:110-118).  Acting uses epsilon = 1 and
evaluation eval_epsilon = 1, so every action is a uniform draw on the sampler's /
evaluator's stream and the replay memory, the episode log and the evaluation returns do
not depend on the network: they pin the schedule itself -- prepopulation, lockstep
t-labels, blocking training events, owner-major flushes, ring eviction, trainer index
draws, counters.  The env keys follow the device executor's per-role derivation
(factory call order: prepopulation, probe, samplers 0..W-1, evaluation).

Output: executor.npz (per case: one 64-bit digest per stored state / next state in
insertion order, actions, rewards, terminals, episode and evaluation events, counters,
the trainer's and the samplers' final PCG64 states).
"""

from __future__ import annotations

import hashlib
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ["PARAQ_BACKEND"] = "numba"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle.envs import SyntheticFrameEnv  # noqa: E402
from paraq import executor as rex  # noqa: E402
from paraq.agent import EpsilonSchedule, HyperParams  # noqa: E402

ROLE_SAMPLER, ROLE_EVAL, ROLE_PREPOP = 1, 3, 4
M64 = (1 << 64) - 1

# (name, mode, W, entry) -- entry "run" = executor.run, "seq" = sequential_reference
CASES = [
    ("both_w8", "both", 8, "run"),
    ("concurrent_w8", "concurrent", 8, "run"),
    ("synchronized_w8", "synchronized", 8, "run"),
    ("standard_w1", "standard", 1, "run"),
    ("standard_w4_seq", "standard", 4, "seq"),
    ("synchronized_w16_seq", "synchronized", 16, "seq"),
]
BASE = dict(C=64, F=4, N=200, batch_size=32, total_steps=192, capacity=300, seed=3,
            eval_period=64, eval_episodes=3, eval_epsilon=1.0, hidden=8)
EPISODE_LENGTH, TERMINAL_P, ACTIONS = 7, 0.05, 18


class FlatFrameEnv(SyntheticFrameEnv):
    """The frame env with flattened uint8 states (the reference MLP's row layout)."""

    @property
    def state_dim(self):
        return int(np.prod(self.state_shape))

    def reset(self, rng):
        return super().reset(rng).reshape(-1)

    def step(self, action, rng):
        s, r, t = super().step(action, rng)
        return s.reshape(-1), r, t


def factory_for(seed: int, W: int):
    keys = ([rex.derived_seed(seed, ROLE_PREPOP, 1), 0]
            + [rex.derived_seed(seed, ROLE_SAMPLER, 1000 + j) for j in range(W)]
            + [rex.derived_seed(seed, ROLE_EVAL, 1000)])
    calls = [0]

    def factory():
        k = keys[calls[0]]
        calls[0] += 1
        return FlatFrameEnv(k, episode_length=EPISODE_LENGTH, action_count=ACTIONS,
                            terminal_p=TERMINAL_P)

    return factory


def digest(a) -> int:
    b = np.ascontiguousarray(np.asarray(a, dtype=np.uint8)).tobytes()
    return int.from_bytes(hashlib.blake2b(b, digest_size=8).digest(), "little")


def pcg_state(rng):
    st = rng.bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    return np.array([s >> 64, s & M64, inc >> 64, inc & M64, st["has_uint32"], st["uinteger"]],
                    dtype=np.uint64)


def run_case(mode: str, W: int, entry: str):
    hp = HyperParams(**BASE, W=W, schedule=EpsilonSchedule(1.0, 1.0, 1)).with_mode(mode)
    captured = []
    orig = rex._Run.__init__

    def init(self, *a, **k):
        orig(self, *a, **k)
        captured.append(self)

    rex._Run.__init__ = init
    try:
        fn = rex.run if entry == "run" else rex.sequential_reference
        rec = fn(hp, factory_for(hp.seed, W))
    finally:
        rex._Run.__init__ = orig
    st = captured[0]
    snap = st.D.snapshot()
    out = {
        "s": np.array([digest(t.state) for t in snap], dtype=np.uint64),
        "s2": np.array([digest(t.next_state) for t in snap], dtype=np.uint64),
        "a": np.array([t.action for t in snap], dtype=np.int64),
        "r": np.array([t.reward for t in snap], dtype=np.float64),
        "term": np.array([t.terminal for t in snap], dtype=bool),
        "version": np.array([st.D.version], dtype=np.int64),
        "episodes": np.array(rec.episodes, dtype=np.float64).reshape(-1, 2),
        "evals": np.array(rec.evals, dtype=np.float64).reshape(-1, 3),
        "events": np.array([f"{s},{k},{v}" for s, k, v in rec.events if k != "theta_hash"]),
        "counter_names": np.array(sorted(rec.counters)),
        "counter_values": np.array([rec.counters[k] for k in sorted(rec.counters)], dtype=np.int64),
        "trainer_pcg": pcg_state(st.trainer_rng),
        "sampler_pcg": np.stack([pcg_state(c.rng) for c in st.ctxs]),
    }
    return out


def main():
    arrays = {}
    for name, mode, W, entry in CASES:
        res = run_case(mode, W, entry)
        for k, v in res.items():
            arrays[f"{name}__{k}"] = v
        print(name, "transitions", len(res["a"]), "episodes", len(res["episodes"]),
              "counters", dict(zip(res["counter_names"], res["counter_values"])))
    np.savez_compressed(os.path.join(HERE, "executor.npz"), **arrays)


if __name__ == "__main__":
    main()
