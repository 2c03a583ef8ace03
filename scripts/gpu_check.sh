cd $GRAFT_REPO_ROOT
for i in 1 2; do for v in 0 2; do
PQ_S2D=$v timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('S2D=$v', [(r['batch'], round(r['us_per_update'],1)) for r in d['learner_batch_sweep']], [(r['W'], round(r['us_per_block'],1)) for r in d['acting_width_sweep']])"
done; done
