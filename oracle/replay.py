"""Replay memory restatement -- TEST INFRASTRUCTURE ONLY (the parity oracle).

Restates the reference ReplayMemory (replay.py:30-93) over frame-stacked uint8
transitions:

* push: append until full, then overwrite the cursor; physical slot of the k-th
  push is k mod capacity; ``version`` counts every push (replay.py:53-59);
* sample: ``rng.integers(0, len, size=B)`` into the physical slot list
  (replay.py:61-66) -- numpy's own PCG64/Lemire, which is the reference algorithm;
* flush: buffers in ascending owner id, each in chronological order
  (replay.py:82-93);
* prepopulate: n uniform-random-action steps on one stream (replay.py:68-80);
* gather: np.stack of states / next states plus the per-field arrays
  (agent.py:76, :100).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Transition:
    state: np.ndarray       # uint8 [4, 84, 84]
    action: int
    reward: float
    next_state: np.ndarray  # uint8 [4, 84, 84]
    terminal: bool          # bootstrap terminal: terminal and not truncated


class ReplayMemory:
    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError("capacity must be at least 1")
        self.capacity = capacity
        self._items: list[Transition] = []
        self._cursor = 0
        self.version = 0

    def __len__(self):
        return len(self._items)

    def push(self, t: Transition) -> None:
        if len(self._items) < self.capacity:
            self._items.append(t)
        else:
            self._items[self._cursor] = t
            self._cursor = (self._cursor + 1) % self.capacity
        self.version += 1

    def sample_indices(self, batch_size: int, rng: np.random.Generator) -> np.ndarray:
        if not self._items:
            raise ValueError("cannot sample from an empty replay memory")
        return rng.integers(0, len(self._items), size=batch_size)

    def sample(self, batch_size: int, rng: np.random.Generator):
        return [self._items[i] for i in self.sample_indices(batch_size, rng)]

    def item(self, slot: int) -> Transition:
        return self._items[slot]

    def flush(self, buffers) -> int:
        moved = 0
        for owner in sorted(buffers):
            for t in buffers[owner]:
                self.push(t)
                moved += 1
            buffers[owner] = []
        return moved

    def prepopulate(self, env, n: int, rng: np.random.Generator) -> None:
        if n > self.capacity:
            raise ValueError("prepopulation count exceeds capacity")
        if n == 0:
            return
        state = env.reset(rng)
        for _ in range(n):
            action = int(rng.integers(env.action_count))
            next_state, reward, terminal = env.step(action, rng)
            boot = terminal and not getattr(env, "truncated", False)
            self.push(Transition(state, action, reward, next_state, boot))
            state = env.reset(rng) if terminal else next_state


def gather(batch):
    """agent.py:76 / :100: stacked states, actions, rewards, next states, terminals."""
    states = np.stack([t.state for t in batch])
    actions = np.asarray([t.action for t in batch], dtype=np.int64)
    rewards = np.asarray([t.reward for t in batch], dtype=np.float64)
    next_states = np.stack([t.next_state for t in batch])
    terminals = np.asarray([t.terminal for t in batch], dtype=bool)
    return states, actions, rewards, next_states, terminals
