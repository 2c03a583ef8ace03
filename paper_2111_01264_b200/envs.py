"""Synthetic 84x84 frame environments on the device (caller side of the hot path).

The frame env is specified in oracle/envs.py (the CPU twin used only by tests):
per step one reward draw and one terminal draw (p = 1/256) on the sampler's PCG64
stream, a fixed horizon that is a time limit (``truncated``), counter-hashed uint8
frames and 4-frame stacks with masked history.  Its state for W samplers lives in
HBM (``DeviceEnvs``) and is advanced by the acting kernel (csrc/env.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .replay import pcg_state_from_generator

TERMINAL_P = 1.0 / 256.0


@dataclass
class FrameEnvSpec:
    """One synthetic frame env, advanced on the GPU (prepopulation / acting)."""

    key: int
    episode_length: int = 200
    action_count: int = 18
    terminal_p: float = TERMINAL_P
    episode: int = -1
    device: bool = True


class DeviceEnvs:
    """HBM state of W synthetic frame envs (pq_envs in include/paraq_b200.h)."""

    def __init__(self, keys, rngs, steps_per_epoch: int):
        torch = N.require_cuda()
        W = len(keys)
        self.W = W
        self.steps = steps_per_epoch
        dev = "cuda"
        self.pcg = torch.from_numpy(
            np.stack([pcg_state_from_generator(r) for r in rngs]).view(np.int64)).to(dev)
        self.episode = torch.full((W,), -1, dtype=torch.int64, device=dev)
        self.t = torch.zeros(W, dtype=torch.int32, device=dev)
        self.stack = torch.full((W, 4), -1, dtype=torch.int32, device=dev)
        self.ep_return = torch.zeros(W, dtype=torch.float64, device=dev)
        self.key = torch.from_numpy(np.asarray(keys, dtype=np.uint64).view(np.int64)).to(dev)
        self.slot_next = torch.zeros(W, dtype=torch.int64, device=dev)
        self.ep_count = torch.zeros(W, dtype=torch.int32, device=dev)
        self.ep_label = torch.zeros((W, steps_per_epoch), dtype=torch.int64, device=dev)
        self.ep_ret = torch.zeros((W, steps_per_epoch), dtype=torch.float64, device=dev)
        self.actions = torch.zeros(W, dtype=torch.int32, device=dev)
        self.reset_next = self.reset_ep = self.reset_slot = None  # compact mode off

    def compact_resets(self) -> None:
        """Compact frame allocation: 1 slot per step per env (slot_next) plus the step's
        reset frames at consecutive sequence numbers from reset_next, in sampler order."""
        torch = N.require_cuda()
        self.reset_next = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.reset_ep = torch.full((self.W,), -1, dtype=torch.int64, device="cuda")
        self.reset_slot = torch.zeros(self.W, dtype=torch.int32, device="cuda")

    def struct(self) -> N.PqEnvs:
        return N.PqEnvs(*(None if getattr(self, f) is None else getattr(self, f).data_ptr()
                          for f, _ in N.PqEnvs._fields_))

    def reset_all(self, slots, ring, stream=None) -> None:
        N.check(N.load().pq_env_reset(self.struct(), self.W, slots.data_ptr(), ring.data_ptr(),
                                      N.stream_ptr(stream)), "env_reset")

    def pcg_states(self) -> np.ndarray:
        return self.pcg.cpu().numpy().view(np.uint64)
