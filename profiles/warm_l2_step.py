"""Eager in-place learner steps (theta_out = theta, opt_out = opt, as the executor runs
them) for a warm-cache ncu pass: with caches not flushed, how much of a step's traffic
reaches DRAM in steady state.  (profiles/one_step.py allocates new theta / opt buffers per
step, so its DRAM bytes are those of a cold optimizer state.)
usage: ncu --cache-control none --metrics dram__bytes_read.sum,... python profiles/warm_l2_step.py [B]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_01264_b200 import _native as N
from paper_2111_01264_b200 import nn as dnn
from paper_2111_01264_b200.envs import FrameEnvSpec
from paper_2111_01264_b200.replay import ReplayMemory

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
mem = ReplayMemory(40000)
mem.prepopulate(FrameEnvSpec(key=5), 40000, np.random.default_rng(1))
theta, target = dnn.init_network(dnn.network_sizes(), 1), dnn.init_network(dnn.network_sizes(), 2)
opt = dnn.OptState.zeros(theta)
ws, cap = dnn.workspace(B, 18)
flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
steps = 20
idx = torch.as_tensor(mem.sample_indices(B * steps, np.random.default_rng(2)), device="cuda")
a = N.PqLearnArgs(theta=theta.struct(), opt=opt.struct(), theta_out=theta.struct(), opt_out=opt.struct(),
                  target=target.struct(), ring=mem.ring.data_ptr(), records=mem.records.data_ptr(),
                  idx=None, idx_base=None, update_counter=None, ext_targets=None, ext_actions=None, n=B,
                  actions=18, gamma=0.99, lr=2.5e-4, rho=0.95, kappa=0.01, nonfinite=flag.data_ptr(),
                  grad_out=None, q_out=None, td_out=None, ws=ws.data_ptr(), max_batch=cap)
for k in range(steps):
    a.idx = idx[k * B:(k + 1) * B].data_ptr()
    N.check(N.load().pq_learn_step(ctypes.byref(a), N.stream_ptr()), "learn_step")
torch.cuda.synchronize()
print(f"B={B}: {steps} in-place steps, flag {int(flag.item())}")
