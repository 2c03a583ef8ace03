"""One persistent-learner launch of K steps after a warm-up launch (for ncu -k
regex:k_learn_persistent -s 1 -c 1).  usage: python profiles/plearn_profile.py [K] [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
C = 4 * 400
hp = HyperParams(C=C, F=4, N=20000, W=8, batch_size=B, total_steps=C, capacity=50000, seed=3,
                 schedule=EpsilonSchedule(0.1, 0.1, 1))
r = DeviceRun(hp, use_graphs=False)
r.begin_epoch(0)
r.learn_run(4)
r.update_counter.zero_()
r.learn_run(K)
torch.cuda.synchronize()
print("done")
