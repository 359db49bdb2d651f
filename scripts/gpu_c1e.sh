cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_march_resident --launch-skip 2 --launch-count 1 \
  -o gpurun_out/c1/resident_fp64 python scripts/profile_c1.py --precision fp64 --ncu --reps 2 > gpurun_out/c1/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/c1/ncu_full.log
