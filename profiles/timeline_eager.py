"""In-situ timeline of one eager learner step at batch B (both translation units' probes:
k_gemm / k_fused / k_head / k_optimizer / k_fc2_partials in qnet.cu, the TMA-engine and
shifted-descriptor kernels in learner.cu).  Per launch: CTA-0 start, dependency release,
last-CTA end (us from the first start), and the kernel's span = last end - release.
usage: python profiles/timeline_eager.py [B]"""
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

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
NAMES = {"G": "k_gemm", "F": "k_fused", "H": "k_head", "O": "k_optimizer", "P": "k_fc2_partials",
         "T": "k_tma_gemm", "D": "k_conv2_dgrad_shift", "S": "k_frames_s2d", "1": "k_conv1_shift",
         "2": "k_conv2_shift", "W": "k_conv1_wgrad_shift", "V": "k_conv2_wgrad_shift", "3": "k_conv3_shift", "4": "k_resident_a", "C": "k_conv3_dgrad_shift", "7": "k_fc1_acc7"}
mem = ReplayMemory(40000)
mem.prepopulate(FrameEnvSpec(key=5), 40000, np.random.default_rng(1))
theta, target = dnn.init_network(dnn.network_sizes(), 1), dnn.init_network(dnn.network_sizes(), 2)
opt = dnn.OptState.zeros(theta)
rng = np.random.default_rng(2)
lib = N.load()
for it in range(5):
    idx = mem.sample_indices(B, rng)
    if it == 4:
        torch.cuda.synchronize()
        lib.pq_timeline(1, None, None)
        lib.pq_timeline_tma(1, None, None)
    theta, opt, _, _, _ = dnn._learn(theta, opt, target, mem.ring, mem.records, idx, B)
torch.cuda.synchronize()
recs = []
for fn in (lib.pq_timeline, lib.pq_timeline_tma):
    out = (ctypes.c_ulonglong * (256 * 12))()
    cnt = ctypes.c_int(0)
    fn(0, ctypes.addressof(out), ctypes.addressof(cnt))
    recs.append(np.array(out).reshape(256, 12)[: cnt.value].astype(np.int64))
t = np.concatenate(recs)
starts = t[[chr(int(r[11])) != "E" for r in t]]
t0 = starts[:, 0].min()
ends = {}
for r in sorted(t, key=lambda x: x[0]):
    if chr(int(r[11])) == "E":
        ends.setdefault((tuple(r[8:11]), int(r[7])), []).append(r[0])
print(f"batch {B}: one eager learner step, us from the first kernel start")
print(f"{'kernel':22s} {'grid':>10s} {'start':>7s} {'release':>8s} {'end':>7s} {'span':>6s}")
for r in sorted(starts, key=lambda x: x[0]):
    tag = chr(int(r[11]))
    q = ends.get((tuple(r[8:11]), ord(tag)), [])
    end = q.pop(0) if q else 0
    rel = r[1] if r[1] > 0 else r[0]
    print(f"{NAMES.get(tag, tag):22s} {str(r[8]) + 'x' + str(r[9]) + 'x' + str(r[10]):>10s} "
          f"{(r[0] - t0) / 1e3:7.1f} {(rel - t0) / 1e3:8.1f} {(end - t0) / 1e3 if end else float('nan'):7.1f} "
          f"{(end - rel) / 1e3 if end else float('nan'):6.1f}")
