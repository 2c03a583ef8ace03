# A/B of learner-step variants at batch 32: eager device time per step (CUDA events)
for v in "PQ_SPLIT_OPT=1" "PQ_SPLIT_OPT=0" "PQ_SPLIT_OPT=1 PQ_PDL=0"; do
  env $v python - <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2111_01264_b200.agent import EpsilonSchedule, HyperParams
from paper_2111_01264_b200.executor import DeviceRun
hp = HyperParams(C=4000, F=4, N=20000, W=8, batch_size=32, total_steps=8000, capacity=50000, seed=3,
                 schedule=EpsilonSchedule(0.1, 0.1, 1))
r = DeviceRun(hp, use_graphs=True, graph_chunk=25)
def ep(e):
    r.flush_and_merge(); r.run_epoch(e); torch.cuda.synchronize()
ep(0)
t0 = time.perf_counter(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); ep(1); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(os.environ.get("PQ_SPLIT_OPT"), os.environ.get("PQ_PDL"), f"epoch {ms:.1f} ms -> {hp.C/ms*1e3:.0f} frames/s, {ms*1e3/(hp.C//hp.F):.1f} us/update")
PY
done
