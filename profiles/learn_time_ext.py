"""Upper bound of moving the target-network forward off the learner's critical path:
batch-32 eager step time with the target forward (groups = 2) vs external TD targets
(groups = 1, the nn.gradient path).  usage: python profiles/learn_time_ext.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2111_01264_b200 import _native as N
from paper_2111_01264_b200 import nn as dnn
from paper_2111_01264_b200.envs import FrameEnvSpec
from paper_2111_01264_b200.replay import ReplayMemory

B = 32
mem = ReplayMemory(40000)
mem.prepopulate(FrameEnvSpec(key=5), 40000, np.random.default_rng(1))
theta, target = dnn.init_network(dnn.network_sizes(), 1), dnn.init_network(dnn.network_sizes(), 2)
opt = dnn.OptState.zeros(theta)
ws, cap = dnn.workspace(B, 18)
flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
steps = 203
idx = torch.as_tensor(mem.sample_indices(B * steps, np.random.default_rng(2)), device="cuda")
tt = torch.zeros(B, device="cuda")
ta = torch.zeros(B, dtype=torch.int32, device="cuda")
for ext in (False, True, False, True):
    a = N.PqLearnArgs(theta=theta.struct(), opt=opt.struct(), theta_out=theta.struct(), opt_out=opt.struct(),
                      target=target.struct(), ring=mem.ring.data_ptr(), records=mem.records.data_ptr(),
                      idx=None, idx_base=None, update_counter=None,
                      ext_targets=tt.data_ptr() if ext else None, ext_actions=ta.data_ptr() if ext else None,
                      n=B, actions=18, gamma=0.99, lr=2.5e-4, rho=0.95, kappa=0.01, nonfinite=flag.data_ptr(),
                      grad_out=None, q_out=None, td_out=None, ws=ws.data_ptr(), max_batch=cap)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(steps):
        if k == 3:
            torch.cuda.synchronize()
            e0.record()
        a.idx = idx[k * B:(k + 1) * B].data_ptr()
        N.check(N.load().pq_learn_step(ctypes.byref(a), N.stream_ptr()), "learn_step")
    e1.record()
    torch.cuda.synchronize()
    print(f"{'external targets (1 network)' if ext else 'target forward (2 networks)'}: "
          f"{e0.elapsed_time(e1) * 1e3 / (steps - 3):.1f} us/step")
