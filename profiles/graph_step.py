"""Untraced CUDA-graph learner step (the bench path, no acting) and the full configs[1]-shaped
epoch (acting + learner streams) of the shipped library, for environment-switch A/B runs.
usage: python profiles/graph_step.py [batch] [capacity]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
hp = HyperParams(C=10000, F=4, N=cap, W=8, batch_size=B, total_steps=100000, capacity=cap, seed=3,
                 schedule=EpsilonSchedule(0.1, 0.1, 1), eval_period=0)
r = DeviceRun(hp, use_graphs=True, graph_chunk=int(os.environ.get("PQ_CHUNK", "25")))


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
t_full = [timed(lambda: full(e)) for e in (2, 3, 4)]
t_learn = [timed(lambda: learn_only(e)) for e in (5, 6, 7)]
r.check_finite()
import hashlib

h = hashlib.sha1(r.theta.master.cpu().numpy().tobytes()).hexdigest()[:12]
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("PQ_"))
print(f"[{tag}] B={B}: full epoch {min(t_full):.1f} ms ({hp.C / min(t_full) * 1e3:.0f} frames/s), "
      f"learner-only {min(t_learn) * 1e3 / r.updates:.2f} us/update, theta {h}")
