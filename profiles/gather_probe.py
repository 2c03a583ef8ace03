"""One 80k-transition replay sample + stack gather per engine (ncu driver for the HBM
roofline of pq_replay_gather: k_gather_tma, then k_gather)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_01264_b200 import _native as N
from paper_2111_01264_b200.envs import FrameEnvSpec
from paper_2111_01264_b200.replay import ReplayMemory, device_pcg, sample_indices_device

mem = ReplayMemory(200_000)
mem.prepopulate(FrameEnvSpec(key=5), 200_000, np.random.default_rng(1))
B = 80_000
idx = sample_indices_device(device_pcg(np.random.default_rng(2)), len(mem), B)
s = torch.empty((B, 4, 84, 84), dtype=torch.uint8, device="cuda")
s2 = torch.empty_like(s)
a = torch.empty(B, dtype=torch.int32, device="cuda")
r = torch.empty(B, dtype=torch.float64, device="cuda")
t = torch.empty(B, dtype=torch.uint8, device="cuda")
for fn in (N.load().pq_replay_gather_tma, N.load().pq_replay_gather_ldg):
    for _ in range(2):
        N.check(fn(mem.ring.data_ptr(), mem.records.data_ptr(), idx.data_ptr(), B, s.data_ptr(), s2.data_ptr(),
                   a.data_ptr(), r.data_ptr(), t.data_ptr(), N.stream_ptr()), "gather")
torch.cuda.synchronize()
print("ok")
