cd $GRAFT_REPO_ROOT
for i in 1 2; do DIST_TC_DEBUG=0 timeout 300 python scripts/tc_debug_timing.py 2>&1 | tail -1; done
