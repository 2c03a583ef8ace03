cd $GRAFT_REPO_ROOT; timeout 60 ./scripts/pdl_event_probe.x
