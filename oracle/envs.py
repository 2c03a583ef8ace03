"""Synthetic 84x84 uint8 frame environment -- TEST INFRASTRUCTURE (CPU side of the
parity pair; paper_2111_01264_b200/csrc/env.cu is the device side).

Modelled on the reference SyntheticLatencyEnv (envs.py:122-174): per step one
reward draw ``rng.random()`` (envs.py:167), a fixed horizon that is a time
limit, i.e. ``truncated`` (envs.py:170-173), and the interface
reset(rng) / step(action, rng) / action_count / truncated.  New for the
Nature-CNN path:

* frames are counter-hashed uint8 84x84 images: 8 pixels per splitmix64 word,
  word p of frame (key, episode, t, a) = splitmix64(base + p) where
  base = splitmix64(splitmix64(splitmix64(key) ^ episode) ^ (t << 8 | a)),
  a = action that produced the frame (255 for a reset frame);
* a true terminal with probability 1/256 per step: a second draw
  ``rng.random() < 1/256`` after the reward draw;
* states are 4-frame stacks [4, 84, 84]; frames before the episode start are
  masked to zero.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
FRAME = 84
STACK = 4
TERMINAL_P = 1.0 / 256.0


def splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _splitmix64_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def frame_base(key: int, episode: int, t: int, action: int) -> int:
    return splitmix64(splitmix64(splitmix64(key) ^ (episode & M64)) ^ (((t << 8) | action) & M64))


def make_frame(key: int, episode: int, t: int, action: int, size: int = FRAME) -> np.ndarray:
    base = frame_base(key, episode, t, action)
    nwords = size * size // 8
    with np.errstate(over="ignore"):
        words = _splitmix64_np(np.uint64(base) + np.arange(nwords, dtype=np.uint64))
    return words.astype("<u8").view(np.uint8).reshape(size, size).copy()


class SyntheticFrameEnv:
    """Frame-stacked synthetic env; deterministic given (key, rng stream, actions)."""

    def __init__(self, key: int, episode_length: int = 200, action_count: int = 18,
                 terminal_p: float = TERMINAL_P, size: int = FRAME):
        if episode_length < 1:
            raise ValueError("episode_length must be at least 1")
        self.key = int(key) & M64
        self.episode_length = episode_length
        self.action_count = action_count
        self.terminal_p = terminal_p
        self.size = size
        self.state_shape = (STACK, size, size)
        self.truncated = False
        self.episode = -1
        self._t = 0
        self._done = True
        self._stack = np.zeros(self.state_shape, dtype=np.uint8)

    def reset(self, rng: np.random.Generator) -> np.ndarray:
        self.episode += 1
        self._t = 0
        self._done = False
        self.truncated = False
        self._stack = np.zeros(self.state_shape, dtype=np.uint8)
        self._stack[-1] = make_frame(self.key, self.episode, 0, 255, self.size)
        return self._stack.copy()

    def step(self, action: int, rng: np.random.Generator):
        if self._done:
            raise RuntimeError("step() after episode end; call reset()")
        if not 0 <= action < self.action_count:
            raise ValueError(f"invalid action {action}")
        reward = float(rng.random())
        true_terminal = bool(rng.random() < self.terminal_p)
        self._t += 1
        frame = make_frame(self.key, self.episode, self._t, int(action), self.size)
        self._stack = np.concatenate([self._stack[1:], frame[None]], axis=0)
        self.truncated = (not true_terminal) and self._t >= self.episode_length
        terminal = true_terminal or self.truncated
        self._done = terminal
        return self._stack.copy(), reward, terminal
