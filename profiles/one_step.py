"""A few eager learner steps on a small replay (profiling driver, not a bench)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2111_01264_b200 import nn as dnn
from paper_2111_01264_b200.envs import FrameEnvSpec
from paper_2111_01264_b200.replay import ReplayMemory

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
mem = ReplayMemory(20000)
mem.prepopulate(FrameEnvSpec(key=1), 10000, np.random.default_rng(0))
theta = dnn.init_network(dnn.network_sizes(), 1)
target = theta.copy()
opt = dnn.OptState.zeros(theta)
rng = np.random.default_rng(1)
for it in range(int(os.environ.get("STEPS", "6"))):
    idx = mem.sample_indices(B, rng)
    theta, opt, _, _, _ = dnn._learn(theta, opt, target, mem.ring, mem.records, idx, B)
torch.cuda.synchronize()
print("ok")
