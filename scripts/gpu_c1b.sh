cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
for p in fp64 fp32; do timeout 300 python scripts/profile_c1.py --precision $p; echo "rc=$?"; done
timeout 900 python -m pytest tests/test_gpu_trace.py tests/test_gpu_edge_cases.py tests/test_gpu_multishape_skip.py tests/test_gpu_reference_suite.py tests/test_gpu_heads.py -q -m gpu -x -p no:cacheprovider > gpurun_out/c1/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c1/pytest.log
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_march_coop --launch-skip 2 --launch-count 1 \
  -o gpurun_out/c1/coop_fp64 python scripts/profile_c1.py --precision fp64 --ncu --reps 2 > gpurun_out/c1/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/c1/ncu_full.log
