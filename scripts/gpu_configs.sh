cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/configs
timeout 1500 python scripts/run_configs.py 2>&1 | grep "^{" | tee gpurun_out/configs/configs.jsonl
