"""Per-CTA trace of the CUDA-graph learner (the bench path) at batch B: for every launch
of one replay of `chunk` steps, the spread of its CTAs' dependency release, accumulator
ready and end times, and where the launch's critical path goes (release -> last end).
usage: python profiles/cta_trace.py [batch] [chunk]"""
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
r.run_epoch(0)
r.flush_and_merge()
r.begin_epoch(1)
gl, nl = r._graphs["learn"]
r.learn_stream.wait_stream(torch.cuda.current_stream())  # the epoch's index table / prologue
lib = N.load()
with torch.cuda.stream(r.learn_stream):
    for _ in range(5):
        gl.replay()
torch.cuda.synchronize()
with torch.cuda.stream(r.learn_stream):  # untraced: learner graph alone, no acting
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(25):
        gl.replay()
    e1.record()
torch.cuda.synchronize()
print(f"untraced learner graph: {e0.elapsed_time(e1) * 1e3 / (25 * nl):.2f} us/step")
out = (ctypes.c_ulonglong * (8192 * 6))()
cnt = ctypes.c_int(0)
lib.pq_cta_trace(1, None, None)
with torch.cuda.stream(r.learn_stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gl.replay()
    e1.record()
torch.cuda.synchronize()
lib.pq_cta_trace(0, ctypes.addressof(out), ctypes.addressof(cnt))
t = np.array(out, dtype=np.uint64).reshape(8192, 6)[: cnt.value]
start, wait, main, end = (t[:, k].astype(np.int64) for k in range(4))
sm = (t[:, 4] >> np.uint64(32)).astype(np.int64)
lin = (t[:, 4] & np.uint64(0xFFFFFFFF)).astype(np.int64)
tag = (t[:, 5] >> np.uint64(48)).astype(np.int64)
part = ((t[:, 5] >> np.uint64(40)) & np.uint64(0xFF)).astype(np.int64)
grid = (t[:, 5] & np.uint64(0xFFFFFFFFFF)).astype(np.int64)
t0 = start.min()
print(f"batch {B}: {cnt.value} CTA records, one replay of {nl} steps, "
      f"{e0.elapsed_time(e1) * 1e3 / nl:.1f} us/step (CUDA events; trace on)")
# launches: consecutive (tag, grid) groups in start order
order = np.argsort(start)
launches = []
cur = None
for i in order:
    key = (int(tag[i]), int(grid[i]))
    if cur is None or cur[0] != key or len(cur[1]) >= key[1]:
        cur = (key, [])
        launches.append(cur)
    cur[1].append(i)
print("launch       ctas | first start | release min/med/max | acc-ready med/max | end med/max | "
      "critical: prev last end -> release min, release -> last end; last CTA (part, sm)")
prev_end = None
for (tg, g), idx in launches:
    idx = np.array(idx)
    rel = lambda x: (x - t0) / 1000.0  # noqa: E731
    w = wait[idx][wait[idx] > 0]
    m = main[idx][main[idx] > 0]
    e = end[idx]
    last = idx[np.argmax(e)]
    gap = f"{(w.min() - prev_end) / 1000:5.1f}" if prev_end is not None and w.size else "    -"
    print(f"{chr(tg)} {g:>4} {len(idx):>5} | {rel(start[idx].min()):6.1f} | "
          + (f"{rel(w.min()):6.1f} {rel(np.median(w)):6.1f} {rel(w.max()):6.1f} | " if w.size else " " * 23 + "| ")
          + (f"{rel(np.median(m)):6.1f} {rel(m.max()):6.1f} | " if m.size else " " * 16 + "| ")
          + f"{rel(np.median(e)):6.1f} {rel(e.max()):6.1f} | {gap} {(e.max() - (w.min() if w.size else start[idx].min())) / 1000:5.1f}"
          + f"  ({part[last]}, {sm[last]})")
    prev_end = e.max()
# per-part breakdown of fused launches
print("\nfused launches by part: ctas, release->acc-ready med/max, acc-ready->end med/max (us)")
for (tg, g), idx in launches[: len(launches) // max(nl, 1)]:
    if chr(tg) != "F":
        continue
    idx = np.array(idx)
    for p in sorted(set(part[idx].tolist())):
        q = idx[part[idx] == p]
        ok = (main[q] > 0) & (wait[q] > 0)
        if not ok.any():
            continue
        a = (main[q][ok] - wait[q][ok]) / 1000
        b = (end[q][ok] - main[q][ok]) / 1000
        print(f"  F{g} part {p}: {len(q):4d} | {np.median(a):5.1f} {a.max():5.1f} | {np.median(b):5.1f} {b.max():5.1f}")
# the update launch (k_opt_tail): part 0 = conv1 blocks (wait for the conv1 weight
# gradient), part 1 = the other parameters (no wait)
print("\nupdate launch by part: ctas, start min/med, release med/max, gradient summed med/max, end med/max "
      "(us from the first record)")
for (tg, g), idx in launches[: len(launches) // max(nl, 1) * 2]:
    if chr(tg) != "T":
        continue
    idx = np.array(idx)
    for p in sorted(set(part[idx].tolist())):
        q = idx[part[idx] == p]
        print(f"  T{g} part {p}: {len(q):4d} | {rel(start[q].min()):6.1f} {rel(np.median(start[q])):6.1f} | "
              f"{rel(np.median(wait[q])):6.1f} {rel(wait[q].max()):6.1f} | "
              + (f"{rel(np.median(main[q])):6.1f} {rel(main[q].max()):6.1f} | " if (main[q] > 0).all() else "   -      -   | ")
              + f"{rel(np.median(end[q])):6.1f} {rel(end[q].max()):6.1f}")
