#!/bin/bash
# Full verification on the GPU box: smoke, GPU tests, default bench (with the CPU
# baseline), the reference arm, an ncu launch list and one full capture of the top kernel.
# usage: scripts/round_verify.sh TAG
TAG=${1:-x}
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --prefill 50000 \
  --capacity 100000 --no-cpu-baseline --no-sweeps > gpurun_out/ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_fused|k_tma_gemm|k_optimizer|k_head" \
  -s 30 -c 10 -o gpurun_out/full_$TAG python profiles/one_step.py > gpurun_out/ncufull_$TAG.log 2>&1
tail -1 gpurun_out/ncufull_$TAG.log
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "cpu", (d.get("cpu_baseline") or {}).get("value"))
print("roofline", json.dumps(d["roofline"]))
print("gather", json.dumps(d["gather_roofline"]))
print("clocks", json.dumps(d["clocks"]))
PY
cat gpurun_out/ref_$TAG.json
