"""A short device-executor run (acting + learner + flush + evaluation), for sanitizers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import run

hp = HyperParams(C=160, F=4, N=400, W=8, batch_size=32, total_steps=320, capacity=2000, seed=5,
                 schedule=EpsilonSchedule(1.0, 0.1, 200), eval_period=0)
rec = run(hp, use_graphs=False)
print("ok", len(rec.epoch_hashes), rec.final_hash)
