"""A few batched Q forwards at width W (ncu driver for the acting forward's launch list).
usage: python scripts/act_fwd.py [W] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_01264_b200 import _native as N
from paper_2111_01264_b200 import nn as dnn

W = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
lib = N.load()
net = dnn.init_network(dnn.network_sizes(18), 3)
ring = torch.randint(0, 256, (4 * W, 84 * 84), dtype=torch.uint8, device="cuda")
refs = torch.arange(4 * W, dtype=torch.int32, device="cuda").view(W, 4)
q = torch.empty((W, 18), dtype=torch.float32, device="cuda")
ws, cap = dnn.workspace(W, 18)
for _ in range(reps):
    N.check(lib.pq_forward(net.struct(), ring.data_ptr(), refs.data_ptr(), None, 4, 0, W, 18, q.data_ptr(),
                           ws.data_ptr(), cap, N.stream_ptr()), "forward")
torch.cuda.synchronize()
print(f"W={W}: {reps} forwards")
