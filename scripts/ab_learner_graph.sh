#!/bin/bash
# untraced learner-graph step time (no acting) of several trees, interleaved: DIR ...
for rep in 1 2; do
  for d in "$@"; do
    (cd $d && echo "$d $(timeout 300 python profiles/cta_trace.py 32 4 2>&1 | grep untraced)")
  done
done
