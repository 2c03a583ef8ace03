"""Per-phase latency of every GEMM CTA-0 in a few eager learner steps (csrc timeline
probes).  Phases: launch->TMEM, wait predecessor, contexts, prologue issue, first MMA,
last MMA, accumulator ready, epilogue done."""
import ctypes
import os
import sys

# the probe build (make probes): the shipped library has no timeline / trace probes
os.environ.setdefault("PQ_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "paper_2111_01264_b200", "_lib", "probes", "libparaq_b200.so"))

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_01264_b200 import _native as N
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
lib = N.load()
out = (ctypes.c_ulonglong * (256 * 12))()
cnt = ctypes.c_int(0)
names = ["F1 conv1", "F2 conv2", "F3 conv3", "F4 fc1", "B4d fc1 dgrad", "B4w fc1 wgrad+rms",
         "B3w conv3 wgrad", "B3d conv3 dgrad", "B2w conv2 wgrad", "B2d conv2 dgrad", "B1w conv1 wgrad"]
for it in range(4):
    idx = mem.sample_indices(B, rng)
    torch.cuda.synchronize()
    lib.pq_timeline(1, None, None)
    theta, opt, _, _, _ = dnn._learn(theta, opt, target, mem.ring, mem.records, idx, B)
    torch.cuda.synchronize()
    lib.pq_timeline(0, ctypes.addressof(out), ctypes.addressof(cnt))
t = np.array(out).reshape(256, 12)[: cnt.value].astype(np.int64)
t0 = t[:, 0].min()
print(f"{cnt.value} GEMM launches (last step); times in us relative to the first launch start")
print("start  tmem  wait  ctx  prol  mma0  mmaN  acc  epi   | durations: tmem wait ctx prol ->mma0 loop accw epi")
for r in sorted(t, key=lambda x: x[0]):
    v = [x for x in r if x > 0]
    rel = [(x - t0) / 1000 for x in v]
    d = np.diff(v) / 1000
    print(" ".join(f"{x:5.1f}" for x in rel), "|", " ".join(f"{x:4.1f}" for x in d))
