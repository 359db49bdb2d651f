cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final1
DIST_TC_DEBUG=0 timeout 300 python scripts/tc_debug_timing.py 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/final1/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/final1/bench.log') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']
print('bench', d['value'], d['ms_per_step'], 'trace', r['trace_ms_per_step'], 'obj', r['objective_ms_per_step'], 'frac', r['frac'], 'e2e', d['e2e']['value'], d['clocks'], d.get('cpu_baseline'))
PY
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/final1/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|^E  " gpurun_out/final1/pytest.log | head -12
timeout 900 python scripts/strong_scaling_probe.py --tile 32 2>&1 | grep "^{" | tee gpurun_out/final1/probe.jsonl
