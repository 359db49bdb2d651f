cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/scale
for t in 32 16; do timeout 900 python scripts/strong_scaling_probe.py --tile $t 2>&1 | grep "^{" | tee -a gpurun_out/scale/probe.jsonl; done
