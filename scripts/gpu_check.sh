cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 200 python profiles/timeline_act.py 512 | head -4
BATCHES="1024" timeout 400 bash scripts/ab_kern.sh 2>&1 | head -2
timeout 200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print([ (r['W'], round(r['us_per_block'],1)) for r in d['acting_width_sweep']]); print([(r['batch'], round(r['us_per_update'],1)) for r in d['learner_batch_sweep']])"
