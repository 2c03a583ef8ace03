# bench builds back to back: DIR:EXTRA_FLAGS ...
run() {
  (cd $1 && timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline $2 2>/tmp/ab_err.txt | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', round(d['value']), round(d['e2e']['value']), d['roofline']['per_launch'])" || tail -3 /tmp/ab_err.txt)
}
for spec in "$@"; do run "${spec%%:*}" "${spec#*:}"; done
