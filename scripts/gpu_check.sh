cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in 0 1; do
PQ_S2DPF=$v timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('PF=$v', [(r['batch'], round(r['us_per_update'],1)) for r in d['learner_batch_sweep']])"
done; done
