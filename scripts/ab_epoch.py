"""Epoch-level A/B: frames/s of the configs[1] epoch with and without the concurrent
acting stream (learner graphs only), 1M-transition replay.  Works on older trees too.
usage: python scripts/ab_epoch.py [capacity]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
hp = HyperParams(C=10000, F=4, N=cap, W=8, batch_size=32, total_steps=60000, capacity=cap, seed=1,
                 schedule=EpsilonSchedule(0.1, 0.1, 1), eval_period=0)
r = DeviceRun(hp, use_graphs=True, graph_chunk=25)


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def full(e):
    r.flush_and_merge()
    r.run_epoch(e)


def learn_only(e):
    r.flush_and_merge()
    r.begin_epoch(e)
    gl, nl = r._graphs["learn"]
    r.learn_stream.wait_stream(torch.cuda.current_stream())  # the epoch's index table / prologue
    with torch.cuda.stream(r.learn_stream):
        for _ in range(r.updates // nl):
            gl.replay()
    torch.cuda.current_stream().wait_stream(r.learn_stream)


full(0)
full(1)
t_full = [timed(lambda: full(e)) for e in (2, 3)]
t_learn = [timed(lambda: learn_only(e)) for e in (4, 5)]
print(f"{os.path.basename(os.getcwd())}: full epoch {min(t_full):.1f} ms ({hp.C / min(t_full) * 1e3:.0f} frames/s), "
      f"learner-only {min(t_learn):.1f} ms ({min(t_learn) * 1e3 / r.updates:.1f} us/update)")
