"""Persistent learner vs the one-shot learner step on identical state: parameter /
moment agreement after K steps, and device time per step of both (CUDA events on the
launching stream).  usage: python profiles/plearn_check.py [K] [B] [ctas]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_01264_b200 import _native as N
from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
if len(sys.argv) > 3:
    N.load().pq_plearn_set_ctas(int(sys.argv[3]))
C = 4 * 400
hp = HyperParams(C=C, F=4, N=20000, W=8, batch_size=B, total_steps=C, capacity=50000, seed=3,
                 schedule=EpsilonSchedule(0.1, 0.1, 1))
r = DeviceRun(hp, use_graphs=False)
r.begin_epoch(0)
torch.cuda.synchronize()
state = [r.theta.master, r.theta.shadow, r.opt.m, r.opt.v, r.update_counter, r.nonfinite]
saved = [t.clone() for t in state]


def restore():
    for t, v in zip(state, saved):
        t.copy_(v)
    torch.cuda.synchronize()


def timed(fn):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


# correctness: K steps both ways
for _ in range(K):
    r.learn_step()
torch.cuda.synchronize()
A = [t.clone() for t in state]
restore()
r.learn_run(K)
torch.cuda.synchronize()
Bv = [t.clone() for t in state]
names = ["master", "shadow", "m", "v", "counter", "nonfinite"]
for nm, x, y, x0 in zip(names, A, Bv, saved):
    if nm in ("counter", "nonfinite"):
        print(f"{nm}: oneshot {x.tolist()} persistent {y.tolist()}")
        continue
    x, y, x0 = x.float(), y.float(), x0.float()
    dx = (x - x0).norm().item()
    err = (x - y).norm().item()
    print(f"{nm}: |oneshot - persistent| = {err:.3e}   |update| = {dx:.3e}   rel {err / max(dx, 1e-30):.3e}   "
          f"max abs {(x - y).abs().max().item():.3e}")
# timing
restore()
n_t = min(200, C // 4)
for _ in range(3):
    restore()
    t1 = timed(lambda: [r.learn_step() for _ in range(n_t)])
    restore()
    t2 = timed(lambda: r.learn_run(n_t))
    print(f"{n_t} steps: one-shot eager {t1 * 1e3 / n_t:.1f} us/step   persistent {t2 * 1e3 / n_t:.1f} us/step")

# per-phase trace of a few steps: max over CTAs of (jobs done - previous barrier release)
G = int(sys.argv[3]) if len(sys.argv) > 3 else torch.cuda.get_device_properties(0).multi_processor_count - 20
steps = 6
nph = 5 + 10 * steps
buf = torch.zeros(nph * G * 4, dtype=torch.int64, device="cuda")
N.load().pq_plearn_trace(buf.data_ptr())
restore()
r.learn_run(steps)
torch.cuda.synchronize()
N.load().pq_plearn_trace(None)
t = buf.view(nph, G, 4).cpu().numpy().astype(np.int64)
rel = t[:, :, 1].min(axis=1)  # first barrier release per phase
spread = t[:, :, 1].max(axis=1) - rel
prev = np.concatenate([[t[0, :, 0].min()], rel[:-1]])
work = t[:, :, 0].max(axis=1) - prev
work_med = np.median(t[:, :, 0] - prev[:, None], axis=1)
bar = rel - t[:, :, 0].max(axis=1)
JOBS = ["F1", "F2", "F3", "F4", "HEAD", "B4D", "OPT_FC2", "B3D", "B3W", "B4W", "B2D", "B2W", "OPT_C3",
        "B1W", "OPT_C2", "OPT_C1", "G1"]
print("phase: work(max CTA) / work(median CTA) / last-arrival->release / release spread [us] | slowest job types")
for k in range(nph):
    lab = f"pro{k}" if k < 5 else f"u{(k - 5) // 10}.P{(k - 5) % 10}"
    typ = t[k, :, 2]
    dur = t[k, :, 3]
    per = {}
    for ty, d in zip(typ, dur):
        if d > 0:
            per.setdefault(JOBS[ty], []).append(d / 1e3)
    desc = " ".join(f"{nm}:{np.median(v):.1f}/{max(v):.1f}" for nm, v in sorted(per.items(), key=lambda kv: -max(kv[1])))
    print(f"{lab:>8}: {work[k] / 1e3:7.2f} {work_med[k] / 1e3:7.2f} {bar[k] / 1e3:6.2f} {spread[k] / 1e3:6.2f} | {desc}")


# per-tile probes of CTA 0: start, accumulator ready, staged, tables, copies done, synced
import ctypes
lib = N.load()
out = (ctypes.c_ulonglong * (256 * 12))()
cnt = ctypes.c_int(0)
restore()
lib.pq_plearn_timeline(1, None, None)
r.learn_run(3)
torch.cuda.synchronize()
lib.pq_plearn_timeline(0, ctypes.addressof(out), ctypes.addressof(cnt))
tt = np.array(out).reshape(256, 12)[: cnt.value].astype(np.int64)
print(f"{cnt.value} CTA-0 tiles; us: mainloop(->acc) ->staged ->tables ->copies ->sync | nk BN")
for row in tt:
    ts = row[:6].astype(np.float64)
    seg = []
    prev = ts[0]
    for k in range(1, 6):
        if ts[k] > 0:
            seg.append(f"{(ts[k] - prev) / 1e3:6.2f}")
            prev = ts[k]
        else:
            seg.append("     -")
    print(" ".join(seg), f"| {row[6]} {row[7]}")
