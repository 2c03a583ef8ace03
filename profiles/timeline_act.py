"""In-situ timeline of one batched Q-inference call (pq_forward, configs[2]) at width W
(probe build, both translation units).  usage: python profiles/timeline_act.py [W]"""
import ctypes
import os
import sys

os.environ.setdefault("PQ_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                             "paper_2111_01264_b200", "_lib", "probes", "libparaq_b200.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_01264_b200 import _native as N
from paper_2111_01264_b200 import nn as dnn

W = int(sys.argv[1]) if len(sys.argv) > 1 else 512
NAMES = {"G": "k_gemm", "F": "k_fused", "H": "k_head", "S": "k_frames_s2d", "1": "k_conv1_shift",
         "2": "k_conv_shift<2>", "3": "k_conv_shift<3>", "4": "k_resident_a", "7": "k_fc1_acc7", "T": "k_tma_gemm"}
lib = N.load()
net = dnn.init_network(dnn.network_sizes(18), 3)
ring = torch.randint(0, 256, (4 * W, 84 * 84), dtype=torch.uint8, device="cuda")
refs = torch.arange(4 * W, dtype=torch.int32, device="cuda").view(W, 4)
q = torch.empty((W, 18), dtype=torch.float32, device="cuda")
ws, cap = dnn.workspace(W, 18)


def go():
    N.check(lib.pq_forward(net.struct(), ring.data_ptr(), refs.data_ptr(), None, 4, 0, W, 18, q.data_ptr(),
                           ws.data_ptr(), cap, N.stream_ptr()), "forward")


for _ in range(5):
    go()
torch.cuda.synchronize()
lib.pq_timeline(1, None, None)
lib.pq_timeline_tma(1, None, None)
go()
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
print(f"W {W}: one batched Q inference, us from the first kernel start")
print(f"{'kernel':22s} {'grid':>10s} {'start':>7s} {'release':>8s} {'end':>7s} {'span':>6s}")
for r in sorted(starts, key=lambda x: x[0]):
    tag = chr(int(r[11]))
    qq = ends.get((tuple(r[8:11]), ord(tag)), [])
    end = qq.pop(0) if qq else 0
    rel = r[1] if r[1] > 0 else r[0]
    print(f"{NAMES.get(tag, tag):22s} {str(r[8]) + 'x' + str(r[9]) + 'x' + str(r[10]):>10s} "
          f"{(r[0] - t0) / 1e3:7.1f} {(rel - t0) / 1e3:8.1f} {(end - t0) / 1e3 if end else float('nan'):7.1f} "
          f"{(end - rel) / 1e3 if end else float('nan'):6.1f}")
