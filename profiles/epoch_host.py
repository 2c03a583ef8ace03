"""Host-side breakdown of one configs[1] epoch as bench.py runs it (flush, target sync,
run_epoch enqueue, GPU wait, finite check, theta hash snapshot) and the GPU-timed epoch.
usage: python profiles/epoch_host.py [capacity]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun
from paper_2111_01264_b200.nn import copy_into

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
hp = HyperParams(C=10000, F=4, N=cap, W=8, batch_size=32, total_steps=100000, capacity=cap, seed=3,
                 schedule=EpsilonSchedule(0.1, 0.1, 1), eval_period=0)
r = DeviceRun(hp, use_graphs=True, graph_chunk=int(os.environ.get("CHUNK", "250")))
parts = {}


def epoch(e, rec):
    t = [time.perf_counter()]
    r.flush_and_merge(); t.append(time.perf_counter())
    copy_into(r.target, r.theta); t.append(time.perf_counter())
    r.run_epoch(e); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    r.check_finite(); t.append(time.perf_counter())
    r.record_epoch_hash((e + 1) * hp.C); t.append(time.perf_counter())
    if rec:
        for k, name in enumerate(("flush", "target", "enqueue", "gpu wait", "finite", "hash")):
            parts.setdefault(name, []).append((t[k + 1] - t[k]) * 1e3)


for e in range(3):
    epoch(e, False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for e in range(3, 8):
    epoch(e, True)
e1.record()
torch.cuda.synchronize()
print(f"GPU-timed epoch {e0.elapsed_time(e1) / 5:.2f} ms; host parts (ms, median): " +
      ", ".join(f"{k} {sorted(v)[2]:.2f}" for k, v in parts.items()))
