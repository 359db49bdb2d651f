cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fluid
timeout 240 python -m pytest tests/test_gpu_fluid.py -q -m gpu -x -p no:cacheprovider > gpurun_out/fluid/pytest.log 2>&1; echo "fluid pytest rc=$?"; grep -E "passed|failed|Error|^E  " gpurun_out/fluid/pytest.log | head -20
