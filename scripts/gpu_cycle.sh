#!/bin/bash
# One build -> measure cycle on the GPU box: GPU tests, a bench line and an ncu launch list.
# usage: scripts/gpu_cycle.sh TAG [bench args...]
TAG=${1:-x}; shift
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/tests_$TAG.log
tail -3 gpurun_out/tests_$TAG.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --prefill 50000 \
  --capacity 100000 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
python profiles/summarize_launches.py gpurun_out/launches_$TAG.csv
if [ -n "$PROFILE_FULL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_optimizer|k_head" \
    -s 60 -c 14 -o gpurun_out/full_$TAG python profiles/one_step.py > gpurun_out/ncufull_$TAG.log 2>&1
  tail -1 gpurun_out/ncufull_$TAG.log
fi
