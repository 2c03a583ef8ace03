cd $GRAFT_REPO_ROOT
timeout 300 python profiles/cta_trace.py 32 4 2>&1 | tail -12
