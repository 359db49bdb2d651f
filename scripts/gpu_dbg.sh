cd $GRAFT_REPO_ROOT
for d in 0 1 2 4; do DIST_TC_DEBUG=$d timeout 300 python scripts/tc_debug_timing.py 2>&1 | tail -1; done
