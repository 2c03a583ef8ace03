#!/bin/bash
# Quick learner-latency cycle on the GPU box: graph timeline of the batch-32 step, the
# headline bench line (no sweeps / CPU arm) and the learner parity + bit-identity tests.
# usage: scripts/perf_cycle.sh TAG [pytest -k expr]
TAG=${1:-x}
K=${2:-"learner or pipelined or fused_backward or executor"}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python profiles/timeline_graph.py 32 4 > gpurun_out/tl_$TAG.txt 2>&1
head -12 gpurun_out/tl_$TAG.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweeps > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print("value", round(d["value"]), "updates/s", round(d["learner_updates_per_s"]), "e2e", round(d["e2e"]["value"]),
      "roofline", d["roofline"]["per_launch"])
PY
timeout 900 python -m pytest tests -q -m gpu -x -k "$K" 2>&1 | tail -3
