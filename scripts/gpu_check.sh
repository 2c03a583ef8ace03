cd $GRAFT_REPO_ROOT; timeout 200 python profiles/cta_trace.py 32 4 2>&1 | tail -14
