cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
for p in fp64 fp32; do timeout 300 python scripts/profile_c1.py --precision $p; echo "rc=$?"; done
timeout 900 python -m pytest tests/test_gpu_narrow.py -q -m gpu -p no:cacheprovider -s > gpurun_out/c1/pytest_narrow.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|C1 iterate|Error|^E " gpurun_out/c1/pytest_narrow.log | head -20
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/c1/pytest_all.log 2>&1; echo "pytest-all rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/c1/pytest_all.log | tail -8
