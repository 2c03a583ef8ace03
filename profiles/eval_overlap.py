"""Cost of the per-epoch evaluation (30 episodes, epsilon 0.05, every 10k steps: the
HyperParams defaults) on a configs[1]-shaped run: wall time of run() with and without it.
usage: python profiles/eval_overlap.py [epochs]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun

E = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for period in (0, 10_000, 0, 10_000):
    hp = HyperParams(C=10000, F=4, N=50_000, W=8, batch_size=32, total_steps=E * 10_000, capacity=100_000,
                     seed=1, schedule=EpsilonSchedule(0.1, 0.1, 1), eval_period=period)
    r = DeviceRun(hp)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rec = r.execute()
    dt = time.perf_counter() - t0
    print(f"eval_period={period}: {dt * 1e3 / E:.1f} ms/epoch wall ({E} epochs, {len(rec.evals)} evals: "
          f"{[round(m, 3) for _, m, _ in rec.evals][:3]})")
