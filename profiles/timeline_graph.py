"""Timeline of the CUDA-graph learner (the bench path): CTA 0 phase stamps of every GEMM
(G), head (H) and optimizer (O) launch of one graph replay of `chunk` learner steps.
GEMM columns: start, predecessor done, contexts, prologue, first MMA, last MMA,
accumulator, epilogue done; H / O: start, predecessor done, end.
usage: python profiles/timeline_graph.py [batch] [chunk]"""
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
from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 4
hp = HyperParams(C=4000, F=4, N=20000, W=8, batch_size=B, total_steps=8000, capacity=50000, seed=3,
                 schedule=EpsilonSchedule(0.1, 0.1, 1), eval_period=0)
r = DeviceRun(hp, use_graphs=True, graph_chunk=chunk)
r.flush_and_merge()
r.run_epoch(0)  # captures the graphs
r.flush_and_merge()
r.begin_epoch(1)
gl, nl = r._graphs["learn"]
r.learn_stream.wait_stream(torch.cuda.current_stream())  # the epoch's index table / prologue
lib = N.load()
with torch.cuda.stream(r.learn_stream):
    for _ in range(5):
        gl.replay()
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * (256 * 12))()
cnt = ctypes.c_int(0)
lib.pq_timeline(1, None, None)
with torch.cuda.stream(r.learn_stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gl.replay()
    e1.record()
torch.cuda.synchronize()
lib.pq_timeline(0, ctypes.addressof(out), ctypes.addressof(cnt))
t = np.array(out).reshape(256, 12)[: cnt.value].astype(np.int64)
t0 = t[:, 0].min()
ends = {}  # (grid, tag) -> end times of the last CTA, in order
for rr in sorted(t, key=lambda x: x[0]):
    if chr(int(rr[11])) == "E":
        ends.setdefault((tuple(rr[8:11]), int(rr[7])), []).append(rr[0])
print(f"batch {B}: {cnt.value} probe records in one replay of {nl} steps, "
      f"{e0.elapsed_time(e1) * 1e3 / nl:.1f} us/step (CUDA events)")
print("tag grid       last-CTA-end | start -> CTA-0 stamps (us from the first start) | durations")
for rr in sorted(t, key=lambda x: x[0]):
    tag = chr(int(rr[11])) if rr[11] else "?"
    if tag == "E":
        continue
    q = ends.get((tuple(rr[8:11]), ord(tag)), [])
    end = f"{(q.pop(0) - t0) / 1000:7.1f}" if q else "      ?"
    v = [x for x in rr[:8] if x > 0]
    rel = [(x - t0) / 1000 for x in v]
    d = np.diff(v) / 1000
    grid = f"{rr[8]}x{rr[9]}x{rr[10]}"
    print(f"{tag} {grid:>10} {end} | " + " ".join(f"{x:6.1f}" for x in rel), "|", " ".join(f"{x:4.1f}" for x in d))
