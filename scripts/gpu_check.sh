cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in 64,0,1 320,2,2; do
 PQ_OPT_TAIL=$v PQ_CHUNK=250 timeout 300 python profiles/graph_step.py 32 2>&1 | tail -1
done; PQ_CHUNK=250 timeout 300 python profiles/graph_step.py 32 2>&1 | tail -1; done
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
