cd $GRAFT_REPO_ROOT; timeout 400 python bench.py --steps 3 --warmup 3 --no-sweeps --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"value\"]), round(d[\"e2e\"][\"value\"]), d[\"roofline\"][\"per_launch\"], d[\"ms_per_step\"])"
