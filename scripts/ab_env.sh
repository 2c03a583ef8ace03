#!/bin/bash
# In-epoch bench A/B of (tree, environment) variants, interleaved twice: "DIR|VAR=1 VAR2=0" ...
run() {
  local dir="${1%%|*}" envs="${1#*|}"
  [ "$envs" = "$1" ] && envs=""
  (cd "$dir" && env $envs timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-sweeps 2>/tmp/ab_err.txt \
    | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$dir [$envs]', round(d['value']), round(d['e2e']['value']), d['roofline']['per_launch'])" \
    || tail -3 /tmp/ab_err.txt)
}
for rep in 1 2; do for spec in "$@"; do run "$spec"; done; done
