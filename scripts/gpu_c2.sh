cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 600 python scripts/run_configs.py --only C2 2>&1 | grep "^{" ; DIST_TC_STEPPED=1 timeout 600 python scripts/run_configs.py --only C2 2>&1 | grep "^{" | sed 's/^/stepped /'; done
