"""Eager learner step time (CUDA events, 20 steps after 3 warm-up) at the given batches.
usage: python profiles/learn_time.py [B ...]"""
import ctypes
import os
import sys

sys.path.insert(0, os.getcwd())  # the tree under test (scripts/ab_learn_time.sh runs it from each tree)
import numpy as np
import torch

from paper_2111_01264_b200 import _native as N
from paper_2111_01264_b200 import nn as dnn
from paper_2111_01264_b200.envs import FrameEnvSpec
from paper_2111_01264_b200.replay import ReplayMemory

mem = ReplayMemory(40000)
mem.prepopulate(FrameEnvSpec(key=5), 40000, np.random.default_rng(1))
for B in [int(x) for x in sys.argv[1:]] or [256, 1024]:
    theta, target = dnn.init_network(dnn.network_sizes(), 1), dnn.init_network(dnn.network_sizes(), 2)
    opt = dnn.OptState.zeros(theta)
    ws, cap = dnn.workspace(B, 18)
    flag = torch.full((1,), 2**31 - 1, dtype=torch.int32, device="cuda")
    steps = 23
    idx = torch.as_tensor(mem.sample_indices(B * steps, np.random.default_rng(2)), device="cuda")
    a = N.PqLearnArgs(theta=theta.struct(), opt=opt.struct(), theta_out=theta.struct(), opt_out=opt.struct(),
                      target=target.struct(), ring=mem.ring.data_ptr(), records=mem.records.data_ptr(),
                      idx=None, idx_base=None, update_counter=None, ext_targets=None, ext_actions=None, n=B,
                      actions=18, gamma=0.99, lr=2.5e-4, rho=0.95, kappa=0.01, nonfinite=flag.data_ptr(),
                      grad_out=None, q_out=None, td_out=None, ws=ws.data_ptr(), max_batch=cap)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    for k in range(steps):
        if k == 3:
            torch.cuda.synchronize()
            h0 = time.perf_counter()
            e0.record()
        a.idx = idx[k * B:(k + 1) * B].data_ptr()
        N.check(N.load().pq_learn_step(ctypes.byref(a), N.stream_ptr()), "learn_step")
    e1.record()
    host_us = (time.perf_counter() - h0) * 1e6 / (steps - 3)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (steps - 3)
    print(f"B={B}: {us:.1f} us/step, {68.26e6 * B / (us * 1e-6) / 1e12:.1f} TFLOP/s, host issue {host_us:.1f} us/step, "
          f"flag {int(flag.item())}")
