"""the UNMODIFIED reference (`paraq.executor.run`, numba backend) timed
at its own bench shapes with its own harness (harness.ablation_grid: every legal mode x W
cell, distinct derived seeds per trial, mean +- std of RunRecord.duration_s).  Runs only
where /root/reference exists (this container); the result is committed as
profiles/r2_reference_paraq_cpu.{json,md}.  Shapes: the `bench` preset over `desk`
(cli.py:409-432: synthetic env, state_dim 32, A 4, B 32, C 500 -> 512 so that every W in 1..8 divides it, F 4, eps 0.1, no eval)
with hidden 256 and the reference's per-step env latency 0 and 250 us; total_steps is
bounded to 4,000 per run (the preset's 200,000 would take hours) and the full-run time
is extrapolated beside the measurement (harness.py:410-426), never substituted."""
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
os.environ["PARAQ_BACKEND"] = "numba"
sys.path.insert(0, "/root/reference/pkg/src")
from paraq.agent import EpsilonSchedule, HyperParams  # noqa: E402
from paraq.harness import ablation_grid, render_runtime_table, to_factor  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TOTAL, FULL, TRIALS = 4096, 200_704, 3
res = {"cores": len(os.sched_getaffinity(0)), "total_steps": TOTAL, "trials": TRIALS,
       "extrapolated_to": FULL, "grids": []}
md = ["# Unmodified reference (paraq, numba) at its own bench shapes\n",
      f"{res['cores']} host cores (survey container), {TRIALS} trials per cell, {TOTAL} steps per run "
      f"(hours at the preset's {FULL} steps in parentheses: x{FULL // TOTAL} extrapolation).\n"]
for lat in (0.0, 250e-6):
    hp = HyperParams(C=512, F=4, N=512, W=4, batch_size=32, total_steps=TOTAL, eval_period=0, capacity=10_000,
                     schedule=EpsilonSchedule(0.1, 0.1, 1), env="synthetic", hidden=256, latency_s=lat,
                     state_dim=32, action_count=4)
    t0 = time.perf_counter()
    table = ablation_grid(hp, [1, 2, 4, 8], TRIALS)
    cells = {f"{m}/{w}": {"mean_s": s.mean, "std_s": s.std, "steps_per_s": TOTAL / s.mean}
             for (m, w), s in table.cells.items()}
    res["grids"].append({"latency_us": lat * 1e6, "cells": cells, "wall_s": time.perf_counter() - t0,
                         "factor_vs_standard_w1": {f"{m}/{w}": v for (m, w), v in to_factor(table).items()}})
    md.append(f"\n## env latency {lat * 1e6:.0f} us\n\n" + render_runtime_table(table, "markdown", FULL / TOTAL))
    best = max(cells.items(), key=lambda kv: kv[1]["steps_per_s"])
    md.append(f"\nfastest cell {best[0]}: {best[1]['steps_per_s']:.0f} env steps/s\n")
    print(md[-2] + md[-1], flush=True)
with open(os.path.join(OUT, "r2_reference_paraq_cpu.json"), "w") as fh:
    json.dump(res, fh, indent=1)
with open(os.path.join(OUT, "r2_reference_paraq_cpu.md"), "w") as fh:
    fh.write("".join(md))
