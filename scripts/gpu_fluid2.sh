cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/fluid
DIST_TC_DEBUG=0 timeout 300 python scripts/tc_debug_timing.py 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fluid/bench.log 2>&1; echo "bench rc=$?"
DIST_TC_STEPPED=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fluid/bench_stepped.log 2>&1; echo "bench stepped rc=$?"
python - <<'PY'
import json
for f in ['gpurun_out/fluid/bench.log','gpurun_out/fluid/bench_stepped.log']:
    l=[x for x in open(f) if x.startswith('{')]
    d=json.loads(l[-1]); r=d['roofline']
    print(f, d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'frac', r['frac'], d['clocks']['sm_mhz'], d['gpu_launches'])
PY
timeout 900 python scripts/strong_scaling_probe.py --tile 32 2>&1 | grep "^{" | tee gpurun_out/fluid/probe.jsonl
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/fluid/pytest_all.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|^E  " gpurun_out/fluid/pytest_all.log | head -12
