cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
for p in fp64 fp32; do timeout 300 python scripts/profile_c1.py --precision $p; done > gpurun_out/c1/profile_c1.jsonl
cat gpurun_out/c1/profile_c1.jsonl
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_march_resident --launch-skip 2 --launch-count 1 \
  -o gpurun_out/c1/resident_reg_fp64 python scripts/profile_c1.py --precision fp64 --ncu --reps 2 > gpurun_out/c1/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c1/launches_resident.csv python scripts/profile_c1.py --precision fp64 --ncu --reps 2 > gpurun_out/c1/ncu.log 2>&1; echo "ncu2 rc=$?"
