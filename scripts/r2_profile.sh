#!/bin/bash
# Round-2 evidence on the GPU box: the default bench line, the reference arm, ncu launch
# list of the bench, ncu --set full of one learner step, ncu DRAM bytes of both gather
# engines, the per-CTA trace of the captured batch-32 learner graph.
TAG=${1:-r2}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -s probes > /dev/null 2>&1  # the probe build (timelines / CTA traces; PQ_LIB selects it)
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; tail -1 gpurun_out/ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --prefill 50000 \
  --capacity 100000 --no-cpu-baseline --no-sweeps > gpurun_out/ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_fused|k_opt_tail|k_head" \
  -s 30 -c 10 -o gpurun_out/full_$TAG python profiles/one_step.py > gpurun_out/ncufull_$TAG.log 2>&1; tail -1 gpurun_out/ncufull_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:k_gather --csv --log-file gpurun_out/gather_$TAG.csv python profiles/gather_probe.py > gpurun_out/ncugather_$TAG.log 2>&1; tail -1 gpurun_out/ncugather_$TAG.log
timeout 300 python profiles/cta_trace.py 32 4 > gpurun_out/cta_trace_$TAG.txt 2>&1
# large batch: in-situ timeline of one eager step (both translation units' probes) and the
# ncu --set full table of one step
timeout 300 python profiles/timeline_eager.py 1024 > gpurun_out/timeline1024_$TAG.txt 2>&1
STEPS=3 timeout 900 ncu --set full --clock-control none -k regex:"^k_" -s 40 -c 20 -o gpurun_out/full1024_$TAG \
  python profiles/one_step.py 1024 > gpurun_out/ncufull1024_$TAG.log 2>&1; tail -1 gpurun_out/ncufull1024_$TAG.log
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "learner", d["roofline"]["per_launch"])
print("gather", round(d["gather_roofline"]["achieved"]))
print("clocks", json.dumps(d["clocks"]))
r = json.load(open("gpurun_out/ref_$TAG.json"))
print("ref", r["value"], r["cpu_baseline"]["cores"], r.get("cpu_replicas"))
PY
