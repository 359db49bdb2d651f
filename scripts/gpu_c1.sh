cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
for p in fp64 fp32; do timeout 300 python scripts/profile_c1.py --precision $p; echo "rc=$?"; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c1/launches_fp64.csv python scripts/profile_c1.py --precision fp64 --ncu --reps 2 > gpurun_out/c1/ncu.log 2>&1; echo "ncu rc=$?"
