cd $GRAFT_REPO_ROOT
TL_MARCH=1 timeout 400 python scripts/tile_timeline.py > gpurun_out/tl_march.log 2>&1
tail -5 gpurun_out/tl_march.log
